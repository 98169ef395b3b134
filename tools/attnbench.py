"""Causal attention fwd (cuDNN) + bwd (ours vs cuDNN) at the Llama-1B block
shape (B=32, S=256, H=32, hd=64, bf16, token-major), CUDA-event timed:
    python tools/attnbench.py            # timings
    python tools/attnbench.py --once     # one fused backward (ncu target)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2603_05500_b200 import _native as N
from paper_2603_05500_b200.trainer import _Attention

B, S, H, hd = 32, 256, 32, 64
q, k, v = (torch.randn((B * S, H * hd), device="cuda").bfloat16().requires_grad_(True) for _ in range(3))
do = torch.randn((B * S, H * hd), device="cuda").bfloat16()
out = _Attention.apply(q, k, v, B, S, H, hd)
lse = out.grad_fn.saved_tensors[4]
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)


def ours():
    N.call("poetx_attention_bwd", B, S, H, hd, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
           do.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), N.stream_ptr())


def cudnn():
    qt, kt, vt = (t.view(B, S, H, hd).transpose(1, 2) for t in (q, k, v))
    o = F.scaled_dot_product_attention(qt, kt, vt, is_causal=True)
    torch.autograd.grad(o, (q, k, v), do.view(B, S, H, hd).transpose(1, 2))


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


if "--once" in sys.argv:
    ours()
    torch.cuda.synchronize()
else:
    print(f"fused backward: {timeit(ours):.1f} us;  cuDNN fwd+bwd (autograd): {timeit(cudnn):.1f} us")
