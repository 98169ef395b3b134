"""Tensor-core merge product (csrc/merge_tc.cu, kernel K9; reference
layer.py:260-273 ``_transformed_base``, blockdiag.py:76-97).

``poetx_merge_tc`` computes blockdiag(G_R) PM blockdiag(G_P) from fp32
factors on bf16 tensor cores with an on-chip hi/lo split of every fp32
operand.  Checked against a float64 torch reference of the same product:

* fp32 output: within 2e-5 * max|ref| -- the hi/lo split keeps ~16 mantissa
  bits per operand, far below the 2^-9 of a single bf16 rounding (a plain
  bf16 product of G would miss this bound by ~100x, asserted below);
* bf16 output: within one bf16 rounding (2^-8 * max|ref|) of the reference;
* POET-XQ input (int8 codes + per-row scales): the same bounds against the
  dequantized weight;
* the layer merge (poetx_layer_merge, which routes BF16 layers with
  b in {128, 256} through this kernel) is covered against the oracle in
  test_gpu_bench_config.py::test_merge_and_materialize_vs_oracle.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2603_05500_b200 import _native as N

    N.lib()
    return N


def factors(nb, b, scale, gen):
    """Near-orthogonal fp32 blocks like CNP outputs: I + skew + its square."""
    q = torch.randn((nb, b, b), generator=gen, dtype=torch.float64) * scale / b ** 0.5
    q = q - q.transpose(1, 2)
    eye = torch.eye(b, dtype=torch.float64)
    return (eye + 2 * q + 2 * q @ q).float()


def reference(g_r, pm, g_p):
    nbr, b, _ = g_r.shape
    m, n = pm.shape
    w = pm.double().view(nbr, b, n)
    w = torch.einsum("sij,sjn->sin", g_r.double(), w).reshape(m, n)
    w = w.view(m, n // b, b)
    return torch.einsum("msj,sjk->msk", w, g_p.double()).reshape(m, n)


def run(N, g_r, g_p, pm=None, codes=None, scales=None, out_f32=True):
    m = g_r.shape[0] * g_r.shape[1]
    n = g_p.shape[0] * g_p.shape[1]
    b = g_r.shape[1]
    out = torch.empty((m, n), dtype=torch.float32 if out_f32 else torch.bfloat16, device="cuda")
    N.call("poetx_merge_tc", m, n, b, g_r.data_ptr(), g_p.data_ptr(), pm.data_ptr() if pm is not None else None,
           codes.data_ptr() if codes is not None else None, scales.data_ptr() if scales is not None else None,
           n, out.data_ptr(), N.F32 if out_f32 else N.BF16, n, N.stream_ptr())
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("m,n,b", [(256, 512, 128), (512, 256, 256), (1024, 768, 256), (384, 1152, 128)])
@pytest.mark.parametrize("scale", [0.05, 0.3])
def test_merge_tc_vs_float64(N, m, n, b, scale):
    gen = torch.Generator().manual_seed(m * 3 + n + b)
    g_r = factors(m // b, b, scale, gen).cuda()
    g_p = factors(n // b, b, scale, gen).cuda()
    pm = (torch.randn((m, n), generator=gen) / m ** 0.5).to(torch.bfloat16).cuda()
    ref = reference(g_r.cpu(), pm.cpu(), g_p.cpu())
    big = float(ref.abs().max())
    got = run(N, g_r, g_p, pm=pm, out_f32=True).double().cpu()
    err = float((got - ref).abs().max())
    assert err <= 2e-5 * big, (err, big)
    # a single bf16 rounding of the factors would not meet that bound
    naive = reference(g_r.cpu().bfloat16().float(), pm.cpu(), g_p.cpu().bfloat16().float())
    assert float((naive - ref).abs().max()) > 10 * err
    got16 = run(N, g_r, g_p, pm=pm, out_f32=False).double().cpu()
    assert float((got16 - ref).abs().max()) <= 2 ** -8 * big


@pytest.mark.parametrize("m,n,b", [(512, 256, 256), (256, 384, 128)])
def test_merge_tc_quantized_base(N, m, n, b):
    gen = torch.Generator().manual_seed(11 + m + n)
    g_r = factors(m // b, b, 0.1, gen).cuda()
    g_p = factors(n // b, b, 0.1, gen).cuda()
    codes = torch.randint(-127, 128, (m, n), generator=gen, dtype=torch.int8)
    scales = torch.rand(m, generator=gen) * 0.01 + 1e-3
    deq = codes.double() * scales.double()[:, None]
    ref = reference(g_r.cpu(), deq, g_p.cpu())
    big = float(ref.abs().max())
    got = run(N, g_r, g_p, codes=codes.cuda(), scales=scales.cuda(), out_f32=True).double().cpu()
    assert float((got - ref).abs().max()) <= 2e-5 * big


def test_merge_tc_identity_factors_return_pm_exactly(N):
    m, n, b = 512, 512, 256
    eye = torch.eye(b).expand(m // b, b, b).contiguous().cuda()
    pm = torch.randn((m, n), device="cuda").to(torch.bfloat16)
    got = run(N, eye, eye.clone(), pm=pm, out_f32=False)
    assert torch.equal(got, pm)


def test_merge_tc_rejects_bad_shapes(N):
    from paper_2603_05500_b200.errors import ConfigError, ShapeError

    g = torch.zeros((1, 64, 64), device="cuda")
    pm = torch.zeros((64, 64), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ShapeError):
        N.call("poetx_merge_tc", 64, 64, 64, g.data_ptr(), g.data_ptr(), pm.data_ptr(), None, None, 64,
               pm.data_ptr(), N.BF16, 64, N.stream_ptr())
    with pytest.raises(ConfigError):
        N.call("poetx_merge_tc", 300, 256, 256, g.data_ptr(), g.data_ptr(), pm.data_ptr(), None, None, 256,
               pm.data_ptr(), N.BF16, 256, N.stream_ptr())
