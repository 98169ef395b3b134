"""Per-kernel device-time breakdown of one training step (CUPTI via
torch.profiler): python tools/profile_step.py [--model llama-1b] [--mb 32]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2603_05500_b200.trainer import Trainer, llama_config

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama-1b")
ap.add_argument("--mb", type=int, default=32)
ap.add_argument("--variant", default="fast")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--rows", type=int, default=40)
args = ap.parse_args()

cfg = llama_config(args.model, variant=args.variant)
tr = Trainer(cfg, args.mb, merge_gap=0)
tok = torch.randint(0, cfg.vocab, (args.mb, cfg.seq + 1), device="cuda")
for _ in range(3):
    tr.step(tok[:, :-1], tok[:, 1:])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(args.steps):
        tr.step(tok[:, :-1], tok[:, 1:])
    torch.cuda.synchronize()
ev = prof.key_averages()
rows = []
total = 0.0
for e in ev:
    t = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    if t > 0 and e.key and not e.key.startswith("aten::") and not e.key.startswith("cuda"):
        rows.append((t / args.steps / 1e3, e.count // args.steps, e.key))
        total += t / args.steps / 1e3
rows.sort(reverse=True)
print(f"device kernel time per step: {total:.2f} ms")
for ms, cnt, key in rows[: args.rows]:
    print(f"{ms:9.3f} ms {100 * ms / total:5.1f}%  x{cnt:<5d} {key[:110]}")
cpu_total = sum(e.cpu_time_total for e in ev if e.key.startswith("aten::")) / args.steps / 1e3
print(f"(aten CPU time per step ~{cpu_total:.1f} ms)")
