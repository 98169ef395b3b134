"""POET-X training throughput benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model llama-1b] [--micro-batch 32] [--variant fast]

One step = one full POET-X pretraining step of the named Llama on synthetic
tokens (forward, backward, data-parallel all-reduce for N>1, global clip +
AdamW on packed skew parameters and dense parameters).  N>1 is launched by
torchrun, one rank per GPU (token-batch data parallelism, weak scaling).

Prints ONE JSON line on rank 0.  ``value`` = tokens/s over all ranks with
the token batches already resident in HBM; ``e2e`` = the same step through
the public Trainer API with the token batch copied from pinned host memory
and the loss read back every step.  ``roofline`` describes the dominant
kernel (the tcgen05 GEMM, timed with CUDA events around every launch on
its stream during an extra profiled pass of the same steps);
``cpu_baseline`` times the CPU oracle (a restatement of the reference's
numpy algorithm) on a bounded sample, rank 0, N=1 only.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "POET-X train tokens/s (Llama-1B, 1/2/4/8 B200), peak HBM/GPU, % TC roofline"
UNIT = "tokens/s"


TRAFFIC_JSON = os.path.join("profiles", "r02", "ncu_gemm_traffic.json")


def gemm_traffic():
    """Per-launch DRAM traffic of the dominant kernel from the committed ncu
    capture of the current kernel (profiles/r02/ncu_gemm_traffic.json,
    tools/ncu_traffic.sh + tools/ncu_traffic_json.py)."""
    try:
        with open(os.path.join(ROOT, TRAFFIC_JSON)) as f:
            return json.load(f)["traffic_bytes_per_launch"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------- CPU arm --


def _cpu_projection(args):
    """Reference-algorithm (oracle port) fwd+bwd+AdamW of one m->n POET-X
    projection at T tokens, fp32, ordered accumulation, one core."""
    m, n, b, T, seed = args
    import numpy as np

    from oracle import poetx_oracle as O

    r = np.random.default_rng(seed)
    base = (r.standard_normal((m, n)) / np.sqrt(m)).astype(np.float32)
    lay = O.OracleLayer(base, b, r.permutation(m).astype(np.int32), r.permutation(n).astype(np.int32))
    lay.q_r[...] = (0.01 * r.standard_normal(lay.q_r.shape)).astype(np.float32)
    lay.q_p[...] = (0.01 * r.standard_normal(lay.q_p.shape)).astype(np.float32)
    x = r.standard_normal((T, m)).astype(np.float32)
    dz = r.standard_normal((T, n)).astype(np.float32)
    t0 = time.perf_counter()
    z, cache = lay.forward(x)
    gr, gp, dx = lay.backward(cache, dz)
    params = {"r": lay.q_r, "p": lay.q_p}
    st_m = {k: np.zeros_like(v) for k, v in params.items()}
    st_v = {k: np.zeros_like(v) for k, v in params.items()}
    O.adamw_step(params, {"r": gr, "p": gp}, st_m, st_v, 0, 1e-3)
    return time.perf_counter() - t0


def cpu_sample(cfg, T=32):
    """Bounded sample: the seven POET-X projections of ONE decoder block of the
    workload at T tokens, one process per projection (host cores in
    parallel).  Extrapolated to the model's layer count -> tokens/s of the
    POET-X path only (attention/head excluded: favours the CPU)."""
    d, f, b = cfg.d, cfg.f, cfg.block
    shapes = [(d, d), (d, d), (d, d), (d, d), (d, f), (d, f), (f, d)]
    jobs = [(m, n, b, T, i) for i, (m, n) in enumerate(shapes)]
    procs = min(len(jobs), os.cpu_count() or 1)
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(procs) as pool:
        times = pool.map(_cpu_projection, jobs)
    wall = time.perf_counter() - t0
    busy = max(times)
    per_block = busy if procs >= len(jobs) else sum(times) / procs
    tok_s = T / (per_block * cfg.layers)
    sample = (f"{cfg.name} POET-X path: 7 projections of one decoder block (b={b}, fp32, ordered "
              f"accumulation as the reference), T={T} tokens fwd+bwd+AdamW, {procs} processes in "
              f"parallel, x{cfg.layers} layers extrapolated; wall {wall:.1f}s")
    return tok_s, procs, sample


def host_info():
    """Host cores and CPU model ("1 core used of N host cores")."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    if model is None:
        try:
            for line in open("/proc/cpuinfo"):
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        except Exception:
            pass
    return {"host_cores": os.cpu_count(), "cpu_model": model}


def _min_of(fn, reps):
    fn()  # warmup
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def cpu_cfg1_split(reps=3):
    """BASELINE.md §4 / configs[0]: single layer 512x512, b=64, k=3, fp32,
    T=1024 on one host core through the oracle port (the reference's
    algorithm and accumulation order, bitwise pinned to it): forward,
    backward fast and mem, adamw_step, merge_and_reinit; min of `reps` after
    one warmup, time.perf_counter."""
    import numpy as np

    from oracle import poetx_oracle as O

    base, fi, fo, q_r, q_p, x, dz = O.cfg1_inputs()
    out = {}
    for variant in ("fast", "mem"):
        lay = O.OracleLayer(base, 64, fi, fo, variant=variant)
        lay.q_r[...] = q_r
        lay.q_p[...] = q_p
        if variant == "fast":
            out["forward_ms"] = 1e3 * _min_of(lambda: lay.forward(x), reps)
        out[f"backward_{variant}_ms"] = 1e3 * _min_of(lambda: lay.backward(lay.forward(x)[1], dz), reps) \
            - out["forward_ms"]
    lay = O.OracleLayer(base, 64, fi, fo)
    lay.q_r[...] = q_r
    lay.q_p[...] = q_p
    z, c = lay.forward(x)
    gr, gp, _ = lay.backward(c, dz)
    params = {"r": lay.q_r.copy(), "p": lay.q_p.copy()}
    m = {k: np.zeros_like(v) for k, v in params.items()}
    v = {k: np.zeros_like(v) for k, v in params.items()}
    out["adamw_step_ms"] = 1e3 * _min_of(lambda: O.adamw_step(params, {"r": gr, "p": gp}, m, v, 1, 1e-3), reps)
    rng = np.random.default_rng(5)
    out["merge_and_reinit_ms"] = 1e3 * _min_of(
        lambda: lay.merge_and_reinit(rng.permutation(512).astype(np.int32), rng.permutation(512).astype(np.int32)),
        reps)
    out["fwd_bwd_fast_tokens_per_s"] = 1024 / ((out["forward_ms"] + out["backward_fast_ms"]) / 1e3)
    out = {k: round(v, 3) for k, v in out.items()}
    out["config"] = "cfg1: 512x512, b=64, k=3, fp32, T=1024; min of %d after 1 warmup; 1 core (oracle port)" % reps
    return out


def ffma_peak_tflops(dev):
    """Measured FP32 CUDA-core peak (8 independent FFMA chains per thread,
    16 CTAs of 256 per SM, best of 5, CUDA events)."""
    import ctypes as C

    import torch

    from paper_2603_05500_b200 import _native as N

    sink = torch.zeros(256, dtype=torch.float32, device=dev)
    fl = C.c_double()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    best = 0.0
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        N.call("poetx_ffma_probe", 1 << 16, sms * 8, sink.data_ptr(), C.byref(fl), N.stream_ptr(dev))
        b.record()
        b.synchronize()
        best = max(best, fl.value / (a.elapsed_time(b) / 1e3) / 1e12)
    return best


def gpu_cfg1(dev, reps=5):
    """configs[0] on the GPU through the drop-in layer API (fp32 parity path,
    CUDA-core FFMA kernels): the same split as cpu_cfg1_split, device time
    (CUDA events), inputs resident; fraction of the measured FFMA peak."""
    import numpy as np
    import torch

    import paper_2603_05500_b200 as P
    from oracle import poetx_oracle as O

    base, fi, fo, q_r, q_p, x, dz = O.cfg1_inputs()
    lay = P.PoetLinearLayer(torch.from_numpy(base), 64, P.Rng.keyed(0, "cfg1"), device=dev)
    lay.set_permutations(P.PermutationMap.from_forward(fi), P.PermutationMap.from_forward(fo))
    lay.q_r.packed.copy_(torch.from_numpy(q_r))
    lay.q_p.packed.copy_(torch.from_numpy(q_p))
    xd, dzd = torch.from_numpy(x).to(dev), torch.from_numpy(dz).to(dev)

    def dev_ms(fn):
        fn()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    out = {"forward_ms": dev_ms(lambda: lay.forward(xd))}
    for variant in ("fast", "mem"):
        lay.variant = variant
        out[f"backward_{variant}_ms"] = dev_ms(lambda: lay.backward(lay.forward(xd)[1], dzd)) - out["forward_ms"]
    lay.variant = "fast"
    z, c = lay.forward(xd)
    g = lay.backward(c, dzd)
    params = {"q_r": lay.q_r.packed.clone(), "q_p": lay.q_p.packed.clone()}
    st = P.adamw_init(params)
    sched = P.ScheduleConfig(base_lr=1e-3, total_steps=100)
    out["adamw_step_ms"] = dev_ms(lambda: P.optim._adamw_launch(
        list(params.values()), [g.q_r, g.q_p], list(st.m.values()), list(st.v.values()), 1e-3, sched, 1))
    rng = P.Rng.keyed(0, "cfg1-merge")
    out["merge_and_reinit_ms"] = dev_ms(lambda: lay.merge_and_reinit(rng))
    flops = 1.552e9  # cfg1 fast fwd+bwd
    tf = flops / ((out["forward_ms"] + out["backward_fast_ms"]) / 1e3) / 1e12
    peak = ffma_peak_tflops(dev)
    out = {k: round(v, 4) for k, v in out.items()}
    out.update({"fwd_bwd_fast_tokens_per_s": round(1024 / ((out["forward_ms"] + out["backward_fast_ms"]) / 1e3), 1),
                "fwd_bwd_fast_tflops": round(tf, 3), "fp32_ffma_peak_tflops": round(peak, 2),
                "frac_of_fp32_peak": round(tf / peak, 4),
                "config": "cfg1 on cuda: fp32 CUDA-core parity path, device time (CUDA events), min of %d" % reps})
    return out


# ------------------------------------------------------------------ clocks --


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.out = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.out.close()
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sms:
            return None
        loaded = [s for s in sms if s > 0.5 * mx] or sms
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ------------------------------------------------------------------ GPU arm --


def flops_per_token(cfg):
    """Algorithmic FLOPs per token of one training step (fast variant)
    (SURVEY §8d): POET-X linears 4mn + 6b(m+n) (+2mn + 2mb mem), causal
    attention 6*S*d per layer, lm_head 6*d*V."""
    d, f, b, S = cfg.d, cfg.f, cfg.block, cfg.seq
    shapes = [(d, d)] * 4 + [(d, f), (d, f), (f, d)]
    lin = 0.0
    for m, n in shapes:
        lin += 4 * m * n + 6 * b * (m + n)
        if cfg.variant == "mem":
            lin += 2 * m * n + 2 * m * b
    lin *= cfg.layers
    return lin, 6.0 * S * d * cfg.layers, 6.0 * d * cfg.vocab


def cnp_flops_per_step(cfg):
    d, f, b = cfg.d, cfg.f, cfg.block
    dims = sum(m + n for m, n in [(d, d)] * 4 + [(d, f), (d, f), (f, d)])
    return 18.0 * b * b * dims * cfg.layers


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2603_05500_b200 as P
    from paper_2603_05500_b200 import _native as N
    from paper_2603_05500_b200.trainer import Trainer, llama_config

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pg = dist.group.WORLD if dist.is_initialized() else None
    cfg = llama_config(args.model, variant=args.variant)
    trainer = Trainer(cfg, args.micro_batch, seed=args.seed, merge_gap=args.merge_gap, device=dev, pg=pg)
    B, S = args.micro_batch, cfg.seq
    gen = torch.Generator().manual_seed(1000 + rank)
    host_batches = [torch.randint(0, cfg.vocab, (B, S + 1), generator=gen).pin_memory() for _ in range(4)]
    dev_batches = [hb.to(dev) for hb in host_batches]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()

    def barrier():
        if pg is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(n, resident: bool, prof: bool = False):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tok_dev = torch.empty((B, S + 1), dtype=torch.int64, device=dev)
        barrier()
        launches0 = N.launch_count()
        start.record()
        for i in range(n):
            if resident:
                tb = dev_batches[i % len(dev_batches)]
            else:
                tok_dev.copy_(host_batches[i % len(host_batches)], non_blocking=True)
                tb = tok_dev
            loss = trainer.step(tb[:, :-1], tb[:, 1:])
            if not resident:
                loss_host.copy_(loss, non_blocking=True)
        stop.record()
        barrier()
        ms = start.elapsed_time(stop)
        launches = N.launch_count() - launches0
        if trainer.graph is not None:
            launches += n * trainer.graph_launches  # kernels inside each graph replay
        if pg is not None:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches

    for i in range(args.warmup):
        trainer.step(dev_batches[i % 4][:, :-1], dev_batches[i % 4][:, 1:])

    # dominant-kernel roofline: CUDA events around each tcgen05 GEMM launch on its
    # stream, during an eager pass of the same steps (host hooks need eager launches)
    # (projection chains serialised for this pass so each launch's duration is its own)
    lib = N.lib()
    lib.poetx_prof_reset()
    lib.poetx_prof_enable(1)
    trainer.model.concurrent = False
    prof_ms, _ = timed(args.steps, resident=True, prof=True)
    trainer.model.concurrent = True
    lib.poetx_prof_enable(0)
    # peak HBM of an eager step (activations + workspaces + optimizer state)
    torch.cuda.reset_peak_memory_stats(dev)
    timed(1, resident=True)
    peak_eager = torch.cuda.max_memory_allocated(dev) / 1e9

    # graph capture of the whole step, NCCL all-reduces included (captured on the
    # capturing stream's dependency chain); --no-graph launches eagerly
    graph_error = None
    if args.graph:
        torch.cuda.empty_cache()  # the graph's private pool replaces the eager cache
        tb = dev_batches[0]
        def agree(ok):  # every rank replays a graph, or none does (matched collectives)
            if pg is None:
                return ok
            flag = torch.tensor([1 if ok else 0], device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            return bool(flag.item())

        try:
            trainer.capture(tb[:, :-1], tb[:, 1:], agree=agree)
        except Exception as e:  # keep measuring (eagerly) rather than lose the run
            graph_error = f"{type(e).__name__}: {e}"[:200]
            trainer.graph = None
            torch.cuda.synchronize()
            torch.cuda.empty_cache()  # release the abandoned graph pool
        args.graph = trainer.graph is not None
    torch.cuda.reset_peak_memory_stats(dev)
    clocks = ClockSampler(local_rank)
    clocks.start()
    ms, launches = timed(args.steps, resident=True)
    clk = clocks.stop()
    peak_alloc = torch.cuda.max_memory_allocated(dev) / 1e9
    peak_res = torch.cuda.max_memory_reserved(dev) / 1e9
    if pg is not None:  # per-GPU peak = max over ranks
        pk = torch.tensor([peak_alloc, peak_res, peak_eager], device=dev, dtype=torch.float64)
        dist.all_reduce(pk, op=dist.ReduceOp.MAX)
        peak_alloc, peak_res, peak_eager = (float(v) for v in pk.tolist())
    e2e_ms, _ = timed(args.steps, resident=False)
    bad = int(trainer.last_bad.item()) if trainer.last_bad is not None else 0
    import ctypes as C

    tot_ms, cnt, flops = C.c_double(), C.c_int64(), C.c_double()
    N.call("poetx_prof_query", b"tc_gemm", C.byref(tot_ms), C.byref(cnt), C.byref(flops))
    k_share = None

    tokens = B * S * world * args.steps
    value = tokens / (ms / 1e3)
    e2e = tokens / (e2e_ms / 1e3)
    hbm, tf_burst, tf_sus, src = peaks()
    lin, attn, head = flops_per_token(cfg)
    step_flops = (lin + attn + head) * B * S + cnp_flops_per_step(cfg)
    step_tc = step_flops * args.steps / (ms / 1e3) / 1e12
    out = None
    if rank == 0:
        achieved = (flops.value / (tot_ms.value / 1e3) / 1e12) if tot_ms.value > 0 else None
        if cnt.value:
            # the kernel's device time per step (its own launches, events on its
            # stream, measured in the eager pass) over the timed step's time; the
            # eager pass itself is slower (one event pair per launch, serialised)
            k_share = tot_ms.value / ms
        out = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic tokens (uniform over vocab 32000), random-init frozen weights",
            "config": {
                "workload": f"{cfg.name} POET-X {cfg.variant} b={cfg.block} k={cfg.neumann_k} pretraining step",
                "micro_batch_per_gpu": B, "seq_len": S, "tokens_per_step_per_gpu": B * S,
                "global_batch": B * world, "parallelism": f"dp{world}",
                "l2": "working set (2.5 GB frozen weights + activations) far larger than the 126 MB L2",
                "merge_gap": args.merge_gap,
                "cuda_graph": bool(args.graph),
                **({"cuda_graph_error": graph_error} if graph_error else {}),
            },
            "peak_hbm_gb": {"eager_step_allocated": round(peak_eager, 2),
                            "timed_allocated": round(peak_alloc, 2), "timed_reserved": round(peak_res, 2),
                            "note": "max over ranks; timed steps replay a CUDA graph whose private pool is in "
                                    "reserved"},
            "step_tc_roofline": {"achieved_tflops": round(step_tc, 1), "peak": tf_sus,
                                 "frac": round(step_tc / tf_sus, 4),
                                 "flops_per_step": step_flops, "peak_source": src + " sustained"},
            "roofline": {
                "kernel": "tc_gemm (tcgen05 mm2 / adjoint)", "bound": "tensor",
                "achieved": round(achieved, 1) if achieved else None, "peak": tf_sus,
                "unit": "TFLOP/s", "frac": round(achieved / tf_sus, 4) if achieved else None,
                "traffic": gemm_traffic(), "traffic_unit": "bytes/launch (ncu dram read+write)",
                "traffic_source": TRAFFIC_JSON, "launches": cnt.value,
                "share_of_step": round(k_share, 4) if k_share else None,
                "kernel_ms_per_step": round(tot_ms.value / args.steps, 3) if cnt.value else None,
                "peak_source": src + " sustained (kernel timed inside a long step)",
                "timing": "CUDA events around every tc_gemm launch on its stream, extra eager profiled pass of the "
                          "same steps with the q/k/v and gate/up chains serialised",
            },
            "e2e": {"value": round(e2e, 1), "unit": UNIT,
                    "h2d_bytes_per_step": B * (S + 1) * 8, "d2h_bytes_per_step": 4},
            "comm_nranks": dist.get_world_size() if pg is not None else 1,
            "gpu_launches": launches,
            "nonfinite_grads": bad,
            "clocks": clk,
        }
    if rank == 0 and world == 1 and not args.no_extras:
        # side measurements after the headline steps (never inside them)
        for key, fn in (("merge", lambda: merge_cost(trainer, ms / args.steps, B * S)),):
            try:
                out[key] = fn()
            except Exception as e:  # reported, never fatal to the headline line
                out[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
        trainer = None  # free the fast trainer (and its graph pool) before the other runs
        import gc

        gc.collect()
        torch.cuda.synchronize(dev)
        N.WORKSPACE.release_all()  # its graph is gone: its pinned workspaces may go too
        torch.cuda.empty_cache()
        for key, fn in (("mem_variant", lambda: mem_variant(args, dev, tf_burst, tf_sus)),
                        ("xq_variant", lambda: mem_variant(args, dev, tf_burst, tf_sus, quantized=True)),
                        ("lora_same_box", lambda: lora_same_box(args, dev)),
                        ("cfg1_gpu", lambda: gpu_cfg1(dev))):
            try:
                out[key] = fn()
            except Exception as e:  # reported, never fatal to the headline line
                out[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
            gc.collect()
            torch.cuda.synchronize(dev)
            N.WORKSPACE.release_all()
            torch.cuda.empty_cache()
        lora, mem = out.get("lora_same_box", {}), out.get("mem_variant", {})
        if "peak_hbm_gb" in lora and "peak_hbm_gb" in mem:
            # the north star's joint target: >= 50% of the tensor-core roofline AND
            # per-GPU peak HBM <= LoRA, both on this box
            out["north_star_check"] = {
                line: {"tc_frac_burst": d["tc_frac_burst"], "peak_hbm_gb": d["peak_hbm_gb"],
                       "peak_le_lora": d["peak_hbm_gb"] <= lora["peak_hbm_gb"], "tc_ge_half_burst": d["tc_frac_burst"] >= 0.5}
                for line, d in (("fast", {"tc_frac_burst": round(step_tc / tf_burst, 4), "peak_hbm_gb": round(peak_eager, 2)}),
                                ("mem", mem))}
            out["north_star_check"]["lora_peak_hbm_gb"] = lora["peak_hbm_gb"]
    return out


def merge_cost(trainer, step_ms, tokens_per_step):
    """Merge-then-reinitialize of the whole model (runner.py:302-327; every
    layer's fp32 CUDA-core CNP, orthogonality audit, keyed permutations, the
    tensor-core merge product K9 and the composite re-permutation), timed with
    CUDA events around Trainer.merge() after the headline steps; the second of
    two merges.  Amortised over the reference default merge_gap of 400 steps."""
    import torch

    times = []
    for _ in range(2):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        trainer.merge()
        e.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(e))
    merge_ms = times[-1]
    gap = 400
    return {"merge_ms": round(merge_ms, 2), "first_merge_ms": round(times[0], 2), "merge_gap": gap,
            "amortised_ms_per_step": round(merge_ms / gap, 3),
            "tokens_per_s_with_merges": round(tokens_per_step / ((step_ms + merge_ms / gap) / 1e3), 1),
            "layers": len(trainer.model.poet_layers()),
            "timing": "CUDA events around Trainer.merge() (eager, host sampling of permutations included)"}


def _timed_steps(step, batches, n):
    import torch

    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for i in range(n):
        tb = batches[i % len(batches)]
        step(tb[:, :-1], tb[:, 1:])
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e)


def mem_variant(args, dev, tf_burst, tf_sus, quantized=False):
    """The same workload with the mem variant (the reference's memory-saving
    layer, layer.py:244-246: no weight-sized activation is saved; t is
    recomputed in backward): CUDA graph, same steps, peak HBM of an eager step
    (allocated) like the headline line's eager figure.  ``quantized``: the
    POET-XQ int8 frozen base (layer.py:169-210, quant.py)."""
    import torch

    from paper_2603_05500_b200.trainer import Trainer, llama_config

    cfg = llama_config(args.model, variant="mem", quantized=quantized)
    tr = Trainer(cfg, args.micro_batch, seed=args.seed, merge_gap=0, device=dev)
    B, S = args.micro_batch, cfg.seq
    gen = torch.Generator().manual_seed(2000)
    batches = [torch.randint(0, cfg.vocab, (B, S + 1), generator=gen).to(dev) for _ in range(4)]
    for i in range(args.warmup):
        tr.step(batches[i % 4][:, :-1], batches[i % 4][:, 1:])
    torch.cuda.reset_peak_memory_stats(dev)
    _timed_steps(tr.step, batches, 1)
    peak = torch.cuda.max_memory_allocated(dev) / 1e9
    torch.cuda.empty_cache()
    tr.capture(batches[0][:, :-1], batches[0][:, 1:])
    ms = _timed_steps(tr.step, batches, args.steps)
    reserved = torch.cuda.max_memory_reserved(dev) / 1e9
    lin, attn, head = flops_per_token(cfg)
    step_flops = (lin + attn + head) * B * S + cnp_flops_per_step(cfg)
    tf = step_flops * args.steps / (ms / 1e3) / 1e12
    bad = int(tr.last_bad.item()) if tr.last_bad is not None else 0
    return {"tokens_per_s": round(B * S * args.steps / (ms / 1e3), 1), "ms_per_step": round(ms / args.steps, 3),
            "achieved_tflops": round(tf, 1), "tc_frac_burst": round(tf / tf_burst, 4),
            "tc_frac_sustained": round(tf / tf_sus, 4), "flops_per_step": step_flops,
            "peak_hbm_gb": round(peak, 2), "graph_reserved_gb": round(reserved, 2), "cuda_graph": tr.graph is not None,
            "nonfinite_grads": bad,
            "flops_note": "mem adds the recomputed t = a PM (2Tmn) and u/a (2Tmb) per layer as algorithmic work (SURVEY §8d)"}


def lora_same_box(args, dev, steps=5):
    """Same-architecture LoRA (frozen bf16 base, rank (b-1)/2 adapters on the
    seven projections, AdamW on the adapters; tools/baselines.py) on this box:
    the peak-HBM and throughput comparator of the north star."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from baselines import BaselineTrainer

    from paper_2603_05500_b200.trainer import llama_config

    cfg = llama_config(args.model, variant="fast")
    # matched trainable parameters: POET-X has (m + n)(b - 1)/2 per linear, LoRA
    # r (m + n); r = b/2 (+0.4%) keeps the adapter GEMMs 16-byte aligned
    rank = cfg.block // 2
    tr = BaselineTrainer(cfg, args.micro_batch, "lora", lora_rank=rank, device=dev)
    B, S = args.micro_batch, cfg.seq
    gen = torch.Generator().manual_seed(3000)
    batches = [torch.randint(0, cfg.vocab, (B, S + 1), generator=gen).to(dev) for _ in range(4)]
    for i in range(3):
        tr.step(batches[i % 4][:, :-1], batches[i % 4][:, 1:])
    torch.cuda.reset_peak_memory_stats(dev)
    ms = _timed_steps(tr.step, batches, steps)
    peak = torch.cuda.max_memory_allocated(dev) / 1e9
    return {"tokens_per_s": round(B * S * steps / (ms / 1e3), 1), "ms_per_step": round(ms / steps, 3),
            "peak_hbm_gb": round(peak, 2), "lora_rank": rank, "trainable_params": tr.trainable,
            "impl": "tools/baselines.py: PyTorch eager, bf16 autocast, fused AdamW"}


def run_reference(args):
    from paper_2603_05500_b200.trainer import llama_config

    cfg = llama_config(args.model, variant=args.variant)
    for _ in range(args.warmup):
        cpu_sample(cfg, T=args.cpu_tokens)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, procs, sample = cpu_sample(cfg, T=args.cpu_tokens)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    return {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "impl": "reference",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * wall / max(1, args.steps), 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name} POET-X {cfg.variant} b={cfg.block} pretraining step (POET-X path sample)",
                   "seq_len": cfg.seq, "parallelism": "host cores"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": sample, **host_info(), "cfg1_split": cpu_cfg1_split()},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(args) -> int:
    """``--gpus N`` (N > 1) outside torchrun: run N ranks on this node, one
    per GPU, exactly as the driver would launch them (torch.distributed.run,
    rendezvous on 127.0.0.1).  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    return subprocess.call(cmd, env=env)


def dry_run(args, rank, world):
    """Launcher check (no GPU work): every rank joins the process group and
    all-reduces its rank; rank 0 prints what the real run would report."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([rank + 1.0])
    if dist.is_initialized():
        dist.all_reduce(t)
    return {"metric": METRIC, "dry_run": True, "n_gpus": world, "gpus_requested": args.gpus,
            "comm_nranks": dist.get_world_size() if dist.is_initialized() else 1,
            "backend": dist.get_backend() if dist.is_initialized() else None,
            "rank_sum": float(t.item())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--model", default="llama-1b")
    ap.add_argument("--micro-batch", type=int, default=32)
    ap.add_argument("--variant", default="fast", choices=("fast", "mem"))
    ap.add_argument("--merge-gap", type=int, default=0, help="0 = no merge inside the timed steps")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-tokens", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the side measurements (mem variant, merge, cfg1) after the headline line's steps")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch eagerly instead of replaying a captured CUDA graph of the step")
    ap.add_argument("--dry-run", action="store_true", help="launcher check only: join the group, no GPU work")
    ap.add_argument("--backend", default=None, help="process-group backend (default nccl; gloo for --dry-run)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(relaunch_under_torchrun(args))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return

    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; reporting the {world} ranks that run",
              file=sys.stderr)
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ  # torchrun, even at N=1
    if distributed:
        import torch
        import torch.distributed as dist

        backend = args.backend or ("gloo" if args.dry_run else "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    if args.dry_run:
        out = dry_run(args, rank, world)
    else:
        out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline and not args.dry_run:
            from paper_2603_05500_b200.trainer import llama_config

            v, procs, sample = cpu_sample(llama_config(args.model, variant=args.variant), T=args.cpu_tokens)
            out["cpu_baseline"] = {"value": round(v, 4), "unit": UNIT, "cores": procs, "kind": "port",
                                   "sample": sample, **host_info(), "cfg1_split": cpu_cfg1_split()}
        print(json.dumps(out), flush=True)
    if distributed:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
