"""RMSNorm + K-gather backward at Llama-1B shape (T = 8192, d = 2048), CUDA
events: python tools/rmsbwdbench.py [K]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
T, d = 8192, 2048
x = torch.randn((T, d), device="cuda").bfloat16()
w = torch.rand(d, device="cuda") + 0.5
rstd = torch.rand(T, device="cuda") + 0.5
dus = [torch.randn((T, d), device="cuda").bfloat16() for _ in range(K)]
inv = [torch.randperm(d, device="cuda").int() for _ in range(K)]
dres = torch.randn((T, d), device="cuda").bfloat16()
dx = torch.empty_like(x)
dw = torch.zeros(d, device="cuda")
ws, wsb = N.workspace(N.lib().poetx_rmsnorm_gather_bwd_workspace_bytes(T, d))
ip = (C.c_void_p * K)(*[t.data_ptr() for t in inv])
dp = (C.c_void_p * K)(*[t.data_ptr() for t in dus])


def run():
    N.call("poetx_rmsnorm_gather_bwd", T, d, x.data_ptr(), w.data_ptr(), rstd.data_ptr(), K, ip, dp,
           dres.data_ptr(), dx.data_ptr(), dw.data_ptr(), 0, ws, wsb, N.stream_ptr())


for _ in range(3):
    run()
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    e.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(e) / 10)
byt = (2 + K + 1) * T * d * 2
print(f"rmsnorm_gather_bwd K={K}: {best * 1e3:.1f} us, {byt / best / 1e9:.2f} TB/s")
