"""Block-diagonal apply / segmented outer at Llama-1B shapes (ncu target):
python tools/blockbench.py apply|outer DIM [transpose]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_05500_b200 as P

op, dim = sys.argv[1], int(sys.argv[2])
tr = len(sys.argv) > 3 and sys.argv[3] == "1"
T, b = 8192, 256
x = torch.randn((T, dim), device="cuda").bfloat16()
y = torch.randn_like(x)
G = P.BlockDiagonalFactor((0.1 * torch.randn((dim // b, b, b), device="cuda")).bfloat16())
def run():
    if op == "apply":
        P.apply_to_features(G, x, transpose=tr)
    else:
        P.segmented_outer(x, y, b)


for _ in range(3):
    run()
torch.cuda.synchronize()
if "--time" in sys.argv:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        run()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    print(f"{op} dim={dim} transpose={int(tr)}: {us:.1f} us, {4 * T * dim / us / 1e3:.0f} GB/s")
