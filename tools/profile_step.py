"""Per-kernel device-time breakdown of one training step (CUPTI via
torch.profiler), grouped by kernel family, against the step's wall time:
python tools/profile_step.py [--model llama-1b] [--mb 32] [--graph]"""
import argparse
import collections
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
ap.add_argument("--graph", action="store_true")
ap.add_argument("--serial", action="store_true", help="no side streams (per-kernel times undisturbed)")
args = ap.parse_args()

FAMILIES = [
    ("tc2_kernel", "tcgen05 pair GEMM (mm2/adjoint/outer/CNP)"),
    ("tc_kernel", "tcgen05 single-CTA GEMM"),
    ("bd_kernel", "block-diagonal apply"),
    ("reduce_splits", "split-T reduce"),
    ("rmsnorm", "rmsnorm+gather"), ("colsum", "rmsnorm+gather"),
    ("swiglu", "swiglu+gather"), ("rope", "rope+scatter"), ("scatter_add", "residual scatter"),
    ("permute", "permute"),
    ("unpack_q", "CNP glue"), ("combine_fwd", "CNP glue"), ("bwd_prep", "CNP glue"), ("pack_dq", "CNP glue"),
    ("to_bf16", "CNP glue"),
    ("adamw", "AdamW+norm"), ("sqdev", "AdamW+norm"),
    ("sdpa", "attention (cuDNN)"), ("cudnn", "attention (cuDNN)"),
    ("nvjet", "lm_head GEMMs (cuBLAS)"), ("SoftMax", "cross-entropy"), ("ce_fwd", "cross-entropy"),
    ("ce_bwd", "cross-entropy"), ("quantize", "POET-XQ"), ("dequant", "POET-XQ"),
]


def family(name):
    for key, fam in FAMILIES:
        if key in name:
            return fam
    return "other torch"


cfg = llama_config(args.model, variant=args.variant)
tr = Trainer(cfg, args.mb, merge_gap=0)
if args.serial:
    tr.model.concurrent = False
tok = torch.randint(0, cfg.vocab, (args.mb, cfg.seq + 1), device="cuda")
for _ in range(3):
    tr.step(tok[:, :-1], tok[:, 1:])
if args.graph:
    tr.capture(tok[:, :-1], tok[:, 1:])
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.record()
    for _ in range(args.steps):
        tr.step(tok[:, :-1], tok[:, 1:])
    e.record()
    torch.cuda.synchronize()
wall = s.elapsed_time(e) / args.steps
kern = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.device_time > 0:
        kern[ev.name][0] += ev.device_time / 1e3 / args.steps
        kern[ev.name][1] += 1
total = sum(v[0] for v in kern.values())
fams = collections.defaultdict(float)
for k, (ms, _) in kern.items():
    fams[family(k)] += ms
print(f"step wall {wall:.2f} ms, kernel time {total:.2f} ms ({100 * total / wall:.1f}%), gaps {wall - total:.2f} ms")
for f, ms in sorted(fams.items(), key=lambda x: -x[1]):
    print(f"  {ms:8.3f} ms {100 * ms / wall:5.1f}%  {f}")
print("top kernels:")
for k, (ms, n) in sorted(kern.items(), key=lambda x: -x[1][0])[: args.rows]:
    print(f"  {ms:8.3f} ms {100 * ms / wall:5.1f}% x{n // args.steps:<5d} {k[:110]}")
