"""One fused int8 GEMM launch (ncu target): python tools/q8one.py M N K transB"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N

M, Nn, K, tb = (int(v) for v in sys.argv[1:5])
a = torch.randn((M, K), device="cuda").bfloat16()
rows, cols = (Nn, K) if tb else (K, Nn)
codes = torch.randint(-127, 128, (rows, cols), device="cuda", dtype=torch.int8)
sc = torch.rand(rows, device="cuda") * 0.01
c = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    N.call("poetx_matmul_q8", M, Nn, K, a.data_ptr(), K, codes.data_ptr(), cols, tb, sc.data_ptr(), c.data_ptr(), Nn,
           N.stream_ptr())
torch.cuda.synchronize()
