"""Host overhead between CUDA-graph steps: Trainer.step() vs bare graph
replays of the same captured step (Llama-1B fast, 32 x 256)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200.trainer import Trainer, llama_config

cfg = llama_config("llama-1b")
tr = Trainer(cfg, 32, merge_gap=0)
tok = torch.randint(0, cfg.vocab, (32, cfg.seq + 1), device="cuda")
for _ in range(2):
    tr.step(tok[:, :-1], tok[:, 1:])
tr.capture(tok[:, :-1], tok[:, 1:])
torch.cuda.synchronize()


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


for rep in range(2):
    a = timed(lambda: tr.step(tok[:, :-1], tok[:, 1:]))
    b = timed(lambda: tr.graph.replay())
    print(f"Trainer.step {a:.3f} ms   bare replay {b:.3f} ms   host overhead {a - b:+.3f} ms")
