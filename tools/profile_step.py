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
ap.add_argument("--quantized", action="store_true")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--rows", type=int, default=40)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--serial", action="store_true", help="no side streams (per-kernel times undisturbed)")
ap.add_argument("--timeline", action="store_true", help="per-stream occupancy: idle gaps, time with one kernel alone")
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
    ("to_bf16", "CNP glue"), ("cnp_fused", "CNP fused (tcgen05)"), ("merge_tc", "merge (tcgen05)"),
    ("adamw", "AdamW+norm"), ("sqdev", "AdamW+norm"),
    ("sdpa", "attention"), ("cudnn", "attention"), ("attn_bwd", "attention"),
    ("nvjet", "lm_head GEMMs (cuBLAS)"), ("SoftMax", "cross-entropy"), ("ce_fwd", "cross-entropy"),
    ("ce_bwd", "cross-entropy"), ("quantize", "POET-XQ"), ("dequant", "POET-XQ"),
]


def family(name):
    for key, fam in FAMILIES:
        if key in name:
            return fam
    return "other torch"


cfg = llama_config(args.model, variant=args.variant, quantized=args.quantized)
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


if args.timeline:
    # kernel intervals per stream from the chrome trace (tid = stream)
    import json
    import tempfile

    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    with open(path) as fh:
        evs = [ev for ev in json.load(fh)["traceEvents"] if ev.get("cat") == "kernel" and ev.get("dur", 0) > 0]

    def tfam(ev):
        # split the pair-GEMM family by grid: full-width launches (mm2 / adjoint /
        # folds / CNP) vs the SM-share-sized segmented outer products
        f = family(ev["name"])
        if "cnp_fused" in ev["name"]:
            f += " fwd" if "true>" in ev["name"] or "1>" in ev["name"] else " bwd"
        if "tc2_kernel" in ev["name"]:
            grid = ev.get("args", {}).get("grid", [0])
            f += " [outer, partial grid]" if grid and grid[0] < 140 else " [full grid]"
        return f
    t0 = min(ev["ts"] for ev in evs)
    t1 = max(ev["ts"] + ev["dur"] for ev in evs)
    edges = []
    for ev in evs:
        edges.append((ev["ts"], 1, ev))
        edges.append((ev["ts"] + ev["dur"], -1, ev))
    edges.sort(key=lambda x: (x[0], x[1]))
    active = {}
    idle = 0.0
    alone = collections.defaultdict(float)
    overl = collections.defaultdict(float)
    by_stream = collections.defaultdict(float)
    last = t0
    gaps = []
    cnp_alone = []
    prev_end = None
    for ts, kind, ev in edges:
        dt = ts - last
        if dt > 0:
            if not active:
                idle += dt
                gaps.append((dt, prev_end["name"][:60] if prev_end else "-", ev["name"][:60]))
            elif len(active) == 1:
                only = next(iter(active.values()))
                alone[tfam(only)] += dt
                if "cnp_fused" in only["name"]:
                    cnp_alone.append((last - t0, dt, tfam(only), prev_end["name"][:50] if prev_end else "-",
                                      f"{ev['name'][:50]} (stream {ev.get('tid')}, cnp on {only.get('tid')})"))
            else:
                for e2 in active.values():
                    overl[tfam(e2)] += dt / len(active)
        last = ts
        if kind > 0:
            active[id(ev)] = ev
            by_stream[ev.get("tid")] += ev["dur"]
        else:
            active.pop(id(ev), None)
            prev_end = ev
    span = (t1 - t0) / 1e3 / args.steps
    print(f"\ntimeline over {args.steps} steps: span {span:.2f} ms/step, idle (no kernel) {idle / 1e3 / args.steps:.2f} ms/step")
    print("largest idle gaps (us: after -> before):")
    for dt, a, b in sorted(gaps, reverse=True)[:12]:
        print(f"  {dt:8.1f}  {a}  ->  {b}")
    print(f"  idle gaps: {len(gaps) / args.steps:.0f} per step, median {sorted(g[0] for g in gaps)[len(gaps) // 2] if gaps else 0:.1f} us")
    print("time with ONE kernel running, by family (ms/step):")
    for f, us in sorted(alone.items(), key=lambda x: -x[1]):
        print(f"  {us / 1e3 / args.steps:8.3f}  {f}")
    print(f"  {sum(alone.values()) / 1e3 / args.steps:8.3f}  total")
    print("CNP kernels running alone (offset in the trace us, duration us, which, last kernel to end before, next edge):")
    for off, dt, f, before, after in sorted(cnp_alone, key=lambda x: -x[1])[:16]:
        print(f"  {off:10.1f} {dt:8.1f}  {f:28s} {before}  ->  {after}")
    print("overlapped time, shared equally among running kernels (ms/step):")
    for f, us in sorted(overl.items(), key=lambda x: -x[1]):
        print(f"  {us / 1e3 / args.steps:8.3f}  {f}")
    print("busy time per stream (ms/step):")
    for sid, us in sorted(by_stream.items(), key=lambda x: -x[1]):
        print(f"  stream {sid}: {us / 1e3 / args.steps:8.3f}")
