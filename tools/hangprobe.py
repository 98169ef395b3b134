"""Repeated eager steps of one config with per-step timing; dumps Python
stacks if a step takes longer than 60 s (diagnosing rare stalls):
python tools/hangprobe.py [model] [mb] [variant] [steps] [--graph]"""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200.trainer import Trainer, llama_config

model, mb, variant, steps = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
cfg = llama_config(model, variant=variant)
tr = Trainer(cfg, mb, merge_gap=0)
tok = torch.randint(0, cfg.vocab, (mb, cfg.seq + 1), device="cuda")
if "--graph" in sys.argv:
    for _ in range(3):
        tr.step(tok[:, :-1], tok[:, 1:])
    tr.capture(tok[:, :-1], tok[:, 1:])
times = []
for i in range(steps):
    faulthandler.dump_traceback_later(60, exit=True)
    t0 = time.perf_counter()
    tr.step(tok[:, :-1], tok[:, 1:])
    torch.cuda.synchronize()
    times.append((time.perf_counter() - t0) * 1e3)
    faulthandler.cancel_dump_traceback_later()
print(" ".join(f"{t:.0f}" for t in times), flush=True)
