"""Where a whole-model merge goes (Trainer.merge, runner.py:302-327):
wall time vs GPU kernel time by kernel family.  python tools/mergeprof.py [model]"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2603_05500_b200.trainer import Trainer, llama_config

name = sys.argv[1] if len(sys.argv) > 1 else "llama-1b"
cfg = llama_config(name)
tr = Trainer(cfg, 8, merge_gap=0)
tok = torch.randint(0, cfg.vocab, (8, cfg.seq + 1), device="cuda")
for _ in range(2):
    tr.step(tok[:, :-1], tok[:, 1:])
tr.merge()
torch.cuda.synchronize()
t0 = time.perf_counter()
tr.merge()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    tr.merge()
    torch.cuda.synchronize()
k = collections.defaultdict(float)
n = collections.Counter()
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.device_time > 0:
        k[ev.name[:60]] += ev.device_time / 1e3
        n[ev.name[:60]] += 1
print(f"{name}: merge wall {wall:.1f} ms, GPU kernel time {sum(k.values()):.1f} ms, {sum(n.values())} kernels")
for nm, ms in sorted(k.items(), key=lambda x: -x[1])[:15]:
    print(f"  {ms:8.2f} ms x{n[nm]:<5d} {nm}")
cpu = collections.defaultdict(float)
for ev in prof.key_averages():
    if ev.cpu_time_total > 0:
        cpu[ev.key[:60]] = ev.cpu_time_total / 1e3
print("top host ops (ms, total incl. children):")
for nm, ms in sorted(cpu.items(), key=lambda x: -x[1])[:12]:
    print(f"  {ms:8.2f}  {nm}")
