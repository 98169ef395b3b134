"""Every mm2 / adjoint GEMM launch of one Llama-1B POET-X step, one launch
per distinct shape (ncu target for the bench roofline's `traffic`):
python tools/gemm_shapes.py [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d, f = 2048, 5632
# (m, n, projections per layer): q/k/v/o, gate/up, down
SHAPES = [(d, d, 4), (d, f, 2), (f, d, 1)]
for m, n, _ in SHAPES:
    a = torch.randn((T, m), device="cuda").bfloat16()
    pm = torch.randn((m, n), device="cuda").bfloat16()
    t = torch.empty((T, n), device="cuda", dtype=torch.bfloat16)
    dt = torch.randn((T, n), device="cuda").bfloat16()
    da = torch.empty((T, m), device="cuda", dtype=torch.bfloat16)
    # mm2: t = a PM ; adjoint: da = dt PM^T
    N.call("poetx_matmul", N.BF16, T, n, m, a.data_ptr(), m, 0, pm.data_ptr(), n, 0, t.data_ptr(), n, 0, N.stream_ptr())
    N.call("poetx_matmul", N.BF16, T, m, n, dt.data_ptr(), n, 0, pm.data_ptr(), n, 1, da.data_ptr(), m, 0,
           N.stream_ptr())
torch.cuda.synchronize()
