"""Fused causal-attention backward (csrc/attention.cu) against the plain
PyTorch fp32 reference of the same op (autograd through explicit softmax
attention), on cuDNN's forward output and logsumexp -- the exact inputs the
trainer hands it."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _reference(q, k, v, do, B, S, H, hd):
    qf, kf, vf = (t.float().view(B, S, H, hd).transpose(1, 2).detach().requires_grad_(True) for t in (q, k, v))
    s = qf @ kf.transpose(-1, -2) / math.sqrt(hd)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
    p = torch.softmax(s.masked_fill(mask, float("-inf")), -1)
    o = (p @ vf).transpose(1, 2).reshape(B * S, H * hd)
    o.backward(do.float())
    return o.detach(), [t.grad.transpose(1, 2).reshape(B * S, H * hd) for t in (qf, kf, vf)]


@pytest.mark.parametrize("B,H", [(2, 4), (1, 32), (3, 8)])
@pytest.mark.parametrize("scale", [1.0, 4.0])
def test_attention_backward_matches_fp32_reference(B, H, scale):
    from paper_2603_05500_b200.trainer import _Attention

    S, hd = 256, 64
    g = torch.Generator("cuda").manual_seed(B * 100 + H + int(scale))
    q, k, v = ((scale * torch.randn((B * S, H * hd), device="cuda", generator=g)).bfloat16().requires_grad_(True)
               for _ in range(3))
    do = torch.randn((B * S, H * hd), device="cuda", generator=g).bfloat16()
    out = _Attention.apply(q, k, v, B, S, H, hd)
    dq, dk, dv = torch.autograd.grad(out, (q, k, v), do)
    o_ref, grads = _reference(q, k, v, do, B, S, H, hd)
    err = (out.float() - o_ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, o_ref.abs().max().item()), err
    for name, got, ref in zip("qkv", (dq, dk, dv), grads):
        err = (got.float() - ref).abs().max().item()
        assert err <= 2e-2 * max(1.0, ref.abs().max().item()), (name, err, ref.abs().max().item())


def test_attention_backward_deterministic():
    from paper_2603_05500_b200.trainer import _Attention

    B, S, H, hd = 2, 256, 8, 64
    g = torch.Generator("cuda").manual_seed(3)
    q, k, v = (torch.randn((B * S, H * hd), device="cuda", generator=g).bfloat16().requires_grad_(True)
               for _ in range(3))
    do = torch.randn((B * S, H * hd), device="cuda", generator=g).bfloat16()
    runs = [torch.autograd.grad(_Attention.apply(q, k, v, B, S, H, hd), (q, k, v), do) for _ in range(2)]
    for a, b in zip(*runs):
        assert torch.equal(a, b)


def test_attention_backward_rejects_other_shapes():
    from paper_2603_05500_b200 import _native as N
    from paper_2603_05500_b200.errors import ConfigError

    x = torch.zeros((512, 128), device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(4 * 512, device="cuda")
    with pytest.raises(ConfigError):
        N.call("poetx_attention_bwd", 1, 512, 1, 128, *(x.data_ptr() for _ in range(5)), lse.data_ptr(),
               *(x.data_ptr() for _ in range(3)), N.stream_ptr())
