"""Single fused row operator at Llama-1B shapes, for ncu captures or CUDA-event
timing: python tools/rowbench.py swiglu_bwd|swiglu|permute [--time]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N

op = sys.argv[1]
T, d, f = 8192, 2048, 5632
st = N.stream_ptr()
vg = torch.randn((T, f), device="cuda").bfloat16()
vu, du, o1, o2 = (torch.randn_like(vg) for _ in range(4))
pf = [torch.randperm(f, device="cuda").int() for _ in range(4)]
def run():
    if op == "swiglu_bwd":
        N.call("poetx_swiglu_gather_bwd", T, f, vg.data_ptr(), vu.data_ptr(), du.data_ptr(), pf[0].data_ptr(),
               pf[1].data_ptr(), pf[2].data_ptr(), pf[3].data_ptr(), o1.data_ptr(), o2.data_ptr(), st)
    elif op == "swiglu":
        N.call("poetx_swiglu_gather", T, f, vg.data_ptr(), vu.data_ptr(), pf[0].data_ptr(), pf[1].data_ptr(),
               o1.data_ptr(), st)
    elif op == "permute":
        N.call("poetx_permute_cols", N.BF16, T, f, pf[0].data_ptr(), vg.data_ptr(), o1.data_ptr(), st)


for _ in range(3):
    run()
torch.cuda.synchronize()
if "--time" in sys.argv:
    nbytes = {"swiglu_bwd": 5, "swiglu": 3, "permute": 2}[op] * T * f * 2
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        run()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    print(f"{op}: {us:.1f} us, {nbytes / us / 1e3:.0f} GB/s")
