"""Does the host keep up between graph replays?  20 trainer.step() calls vs
20 bare graph.replay() calls (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2603_05500_b200.trainer import Trainer, llama_config

cfg = llama_config("llama-1b")
tr = Trainer(cfg, 32, merge_gap=0)
tok = torch.randint(0, cfg.vocab, (32, cfg.seq + 1), device="cuda")
for _ in range(3):
    tr.step(tok[:, :-1], tok[:, 1:])
tr.capture(tok[:, :-1], tok[:, 1:])
for _ in range(3):
    tr.step(tok[:, :-1], tok[:, 1:])
torch.cuda.synchronize()


def timed(fn, n=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


a = timed(lambda: tr.step(tok[:, :-1], tok[:, 1:]))
b = timed(lambda: tr.graph.replay())
c = timed(lambda: tr.step(tok[:, :-1], tok[:, 1:]))
print(f"step {a:.3f} ms, bare replay {b:.3f} ms, step {c:.3f} ms")
