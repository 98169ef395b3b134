"""Throughput and peak HBM for every BASELINE.json config on one B200, with
same-box AdamW and LoRA baselines of the same architecture:

    python tools/configs_bench.py            # all cases, one subprocess each
    python tools/configs_bench.py --one NAME # a single case (JSON line)

POET-X cases run through the Trainer (eager launches so peak memory is
comparable with the eager PyTorch baselines).  Peak HBM = max_memory_allocated
over warmup + timed steps.  Synthetic tokens, random-init weights."""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    "cfg1-layer": dict(kind="layer"),
    "60m-poetx": dict(kind="poet", model="llama-60m", mb=32),
    "60m-adamw": dict(kind="adamw", model="llama-60m", mb=32),
    "60m-lora": dict(kind="lora", model="llama-60m", mb=32, rank=32),
    "350m-poetx-merge5": dict(kind="poet", model="llama-350m", mb=32, merge_gap=5),
    "350m-poetx": dict(kind="poet", model="llama-350m", mb=32),
    "1b-poetx-fast": dict(kind="poet", model="llama-1b", mb=32),
    "1b-poetx-mem": dict(kind="poet", model="llama-1b", mb=32, variant="mem"),
    "1b-poetxq-mem": dict(kind="poet", model="llama-1b", mb=32, variant="mem", quantized=True),
    "1b-adamw": dict(kind="adamw", model="llama-1b", mb=32),
    "1b-lora": dict(kind="lora", model="llama-1b", mb=32, rank=128),
    "8b-poetx-fast": dict(kind="poet", model="llama-8b", mb=1),
    "8b-poetx-mem": dict(kind="poet", model="llama-8b", mb=1, variant="mem"),
    "8b-poetxq-mem": dict(kind="poet", model="llama-8b", mb=1, variant="mem", quantized=True),
    "8b-adamw": dict(kind="adamw", model="llama-8b", mb=1),
    "8b-lora": dict(kind="lora", model="llama-8b", mb=1, rank=128),
    "8b-poetx-fast-mb8": dict(kind="poet", model="llama-8b", mb=8),
}


def timed_steps(step, toks, warmup, steps):
    """(mean, median) per-step time (CUDA events around each eager step, Python
    GC paused).  The mean includes everything (merge steps too); eager
    host-side stalls (allocator) show up as isolated slow steps, which the
    median ignores."""
    import gc
    import statistics

    import torch

    for i in range(warmup):
        step(toks[i % len(toks)])
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    gc.disable()
    try:
        for i in range(steps):
            ev[i][0].record()
            step(toks[i % len(toks)])
            ev[i][1].record()
        torch.cuda.synchronize()
    finally:
        gc.enable()
    ts = [a.elapsed_time(b) for a, b in ev]
    return sum(ts) / len(ts), statistics.median(ts)


def run_layer():
    """BASELINE configs[0]: single POET-X linear 512x512, b=64, k=3, fp32,
    8x128 tokens, fwd+bwd+AdamW through the drop-in layer API, vs the CPU
    oracle on the same shapes."""
    import numpy as np
    import torch

    import paper_2603_05500_b200 as P
    from oracle import poetx_oracle as O

    m = n = 512
    b, T = 64, 1024
    r = np.random.default_rng(0)
    base = (r.standard_normal((m, n)) / np.sqrt(m)).astype(np.float32)
    # a torch-constructed layer keeps device state (numpy-constructed ones mirror
    # the reference's numpy attributes and copy in and out every call)
    lay = P.PoetLinearLayer(torch.from_numpy(base), b, P.Rng.keyed(0, "cfg1"))
    lay.q_r.packed.normal_(0, 0.01)
    lay.q_p.packed.normal_(0, 0.01)
    x = torch.randn((T, m), device="cuda")
    dz = torch.randn((T, n), device="cuda")
    params = {"q_r": lay.q_r.packed, "q_p": lay.q_p.packed}
    st = P.adamw_init(params)
    sched = P.ScheduleConfig(base_lr=1e-3, total_steps=100)

    def step(_):
        z, c = lay.forward(x)
        g = lay.backward(c, dz)
        P.adamw_step(params, {"q_r": g.q_r, "q_p": g.q_p}, st, 1e-3, sched)

    ms, _ = timed_steps(step, [None], 5, 50)
    ref = O.OracleLayer(base, b, lay.perm_in.forward, lay.perm_out.forward)
    xn, dzn = x.cpu().numpy(), dz.cpu().numpy()
    t0 = time.perf_counter()
    zr, cr = ref.forward(xn)
    ref.backward(cr, dzn)
    cpu_s = time.perf_counter() - t0
    flops = 4 * T * m * n + 6 * T * b * (m + n) + 18 * b * b * (m + n)
    return {"tokens_per_s": T / (ms / 1e3), "ms_per_step": ms, "gflops_per_s": flops / (ms / 1e3) / 1e9,
            "cpu_oracle_tokens_per_s": T / cpu_s, "cpu_oracle_s": cpu_s, "cpu_cores": 1,
            "dtype": "f32", "peak_hbm_gb": torch.cuda.max_memory_allocated() / 1e9}


def run_model(c):
    import torch

    from paper_2603_05500_b200.trainer import Trainer, llama_config

    cfg = llama_config(c["model"], variant=c.get("variant", "fast"), quantized=c.get("quantized", False))
    mb = c["mb"]
    g = torch.Generator().manual_seed(0)
    toks = [torch.randint(0, cfg.vocab, (mb, cfg.seq + 1), generator=g).cuda() for _ in range(2)]
    torch.cuda.reset_peak_memory_stats()
    if c["kind"] == "poet":
        tr = Trainer(cfg, mb, merge_gap=c.get("merge_gap", 0))
        trainable = tr.model.poet.numel + tr.model.dense.numel
        step = lambda t: tr.step(t[:, :-1], t[:, 1:])  # noqa: E731
    else:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from baselines import BaselineTrainer

        tr = BaselineTrainer(cfg, mb, c["kind"], c.get("rank", 0))
        trainable = tr.trainable
        step = lambda t: tr.step(t[:, :-1], t[:, 1:])  # noqa: E731
    static_gb = torch.cuda.memory_allocated() / 1e9
    ms, med = timed_steps(step, toks, 3, 15)
    return {"model": cfg.name, "variant": cfg.variant if c["kind"] == "poet" else None,
            "int8_base": bool(c.get("quantized", False)), "micro_batch": mb,
            "seq": cfg.seq, "tokens_per_step": mb * cfg.seq, "tokens_per_s": mb * cfg.seq / (ms / 1e3),
            "ms_per_step": ms, "tokens_per_s_median_step": mb * cfg.seq / (med / 1e3),
            "peak_hbm_gb": torch.cuda.max_memory_allocated() / 1e9, "static_hbm_gb": static_gb, "trainable_params": int(trainable),
            "merge_gap": c.get("merge_gap", 0), "lora_rank": c.get("rank")}


def one(name):
    import torch

    c = CASES[name]
    out = {"case": name, "kind": c["kind"], "gpu": torch.cuda.get_device_name(0)}
    try:
        out.update(run_layer() if c["kind"] == "layer" else run_model(c))
    except torch.OutOfMemoryError as e:
        out["oom"] = str(e).split("\n")[0][:200]
        out["peak_hbm_gb"] = torch.cuda.max_memory_allocated() / 1e9
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--one")
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.one:
        one(a.one)
        return
    lines = []
    for name in a.cases.split(","):
        r = subprocess.run([sys.executable, __file__, "--one", name], capture_output=True, text=True, timeout=900)
        line = next((ln for ln in r.stdout.splitlines() if ln.startswith("{")), None)
        if line is None:
            line = json.dumps({"case": name, "error": (r.stderr or "")[-400:]})
        print(line, flush=True)
        lines.append(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
