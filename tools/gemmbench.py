"""One tcgen05 GEMM launch at a Llama-1B mm2 shape (ncu target):
python tools/gemmbench.py [M N K transB pair]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N

M, Nn, K, tb, pair = (int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (8192, 5632, 2048, 0, 1)))
N.lib().poetx_set_gemm_pair_enabled(pair)
a = torch.randn((M, K), device="cuda").bfloat16()
b = torch.randn((Nn, K) if tb else (K, Nn), device="cuda").bfloat16()
c = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, b.data_ptr(), b.shape[1], tb, c.data_ptr(), Nn, 0,
           N.stream_ptr())
torch.cuda.synchronize()
