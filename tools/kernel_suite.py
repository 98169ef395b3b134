"""One launch of every hot-path kernel family at Llama-1B shapes (T = 8192
tokens, b = 256), each preceded by NVTX-free warm-up, as an ncu target:

    ncu --set full -o gpurun_out/suite python tools/kernel_suite.py
    python tools/kernel_suite.py --summary gpurun_out/suite.ncu-rep > profiles/r01/ncu_kernels.md
or, without a (large) report file:
    ncu --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
        sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --log-file suite.csv \
        python tools/kernel_suite.py
    python tools/kernel_suite.py --summary suite.csv

The summary converts each kernel's ncu duration into achieved TFLOP/s or
GB/s from its ALGORITHMIC work and divides by the measured
peaks (MEASURED_PEAKS.json)."""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

T, d, f, b = 8192, 2048, 5632, 256
NB = 3696  # POET-X blocks of Llama-1B

# kernel-name substring, label, work kind, algorithmic work (FLOP or bytes), in launch order
PLAN = [
    ("tc2_kernel", "mm2 t = a PM (2048->5632)", "flop", 2.0 * T * d * f),
    ("tc2_kernel", "adjoint da = dt PM^T (5632->2048)", "flop", 2.0 * T * d * f),
    ("tc2_kernel", "segmented outer dG (T x 5632, b=256)", "bytes", 2.0 * T * f * 2),
    ("reduce_splits", "split-T reduce (22 blocks)", "bytes", 4.0 * 22 * b * b * 4),
    ("bd_kernel", "block-diagonal apply (T x 5632)", "bytes", 2.0 * T * f * 2),
    ("bd_kernel", "block-diagonal apply^T (T x 2048)", "bytes", 2.0 * T * d * 2),
    ("permute_cols_t8", "feature permutation (T x 2048)", "bytes", 2.0 * T * d * 2),
    ("unpack_q", "CNP unpack (1024 blocks)", "bytes", 1024 * (b * (b - 1) / 2 * 4 + b * b * 2)),
    ("tc2_kernel", "CNP Q^2 (1024 blocks)", "flop", 2.0 * 1024 * b ** 3),
    ("tc2_kernel", "CNP [Q^3|Q^4] (1024 blocks)", "flop", 4.0 * 1024 * b ** 3),
    ("combine_fwd", "CNP combine (1024 blocks)", "bytes", 1024 * b * b * 2 * 5.0),
    ("sqdev_partial", "global grad norm (120.6M params)", "bytes", 120.64e6 * 4),
    ("adamw_kernel", "AdamW + clip (120.6M params)", "bytes", 120.64e6 * 28),
    ("swiglu_gather_bwd", "SwiGLU+gathers backward (T x 5632)", "bytes", 5.0 * T * f * 2),
    ("rmsnorm_gather_bwd", "RMSNorm+3 gathers backward (T x 2048)", "bytes", 6.0 * T * d * 2),
    ("rmsnorm_gather_t8", "RMSNorm+3 gathers forward, 8-token tiles (T x 2048)", "bytes", 4.0 * T * d * 2),
    ("rope_scatter_kernel", "RoPE + output scatter (T x 2048)", "bytes", 2.0 * T * d * 2),
    ("attn_bwd", "causal attention backward (B=32, S=256, H=32, hd=64)", "flop", 32 * 32 * 3 * 10.0 * 128 * 128 * 64),
]


def run():
    import torch

    import paper_2603_05500_b200 as P
    from paper_2603_05500_b200 import _native as N
    from paper_2603_05500_b200.trainer import PoetStack, _ptrs

    st = N.stream_ptr()
    dev = torch.device("cuda")
    a = torch.randn((T, d), device=dev).bfloat16()
    pm = torch.randn((d, f), device=dev).bfloat16()
    t = torch.empty((T, f), device=dev, dtype=torch.bfloat16)
    dt = torch.randn((T, f), device=dev).bfloat16()
    da = torch.empty((T, d), device=dev, dtype=torch.bfloat16)
    N.call("poetx_matmul", N.BF16, T, f, d, a.data_ptr(), d, 0, pm.data_ptr(), f, 0, t.data_ptr(), f, 0, st)
    N.call("poetx_matmul", N.BF16, T, d, f, dt.data_ptr(), f, 0, pm.data_ptr(), f, 1, da.data_ptr(), d, 0, st)
    P.segmented_outer(t, dt, b)  # tc2_kernel + reduce_splits
    G5 = P.BlockDiagonalFactor((0.1 * torch.randn((f // b, b, b), device=dev)).bfloat16())
    G2 = P.BlockDiagonalFactor((0.1 * torch.randn((d // b, b, b), device=dev)).bfloat16())
    P.apply_to_features(G5, t)
    P.apply_to_features(G2, a, transpose=True)
    P.permute_features(a, P.sample_permutation(d, P.Rng(1)), "inverse")
    stack = PoetStack([("all", 1024)], b, dev)
    stack.group.param.normal_(0, 0.01)
    stack.forward_factors()  # unpack, Q^2, [Q^3|Q^4], combine
    n = int(120.64e6)
    p_, g_, m_, v_ = (torch.randn(n, device=dev) * 1e-3 for _ in range(4))
    v_.abs_()
    sched = P.ScheduleConfig(base_lr=1e-3, total_steps=100)
    P.fused_clip_adamw([([p_], [g_], [m_], [v_], 1e-3, 1)], 1.0, sched)  # sqdev + adamw
    vg, vu, du = (torch.randn((T, f), device=dev).bfloat16() for _ in range(3))
    perms = [torch.randperm(f, device=dev).int() for _ in range(4)]
    o1, o2 = torch.empty_like(vg), torch.empty_like(vg)
    N.call("poetx_swiglu_gather_bwd", T, f, vg.data_ptr(), vu.data_ptr(), du.data_ptr(), *[q.data_ptr() for q in perms],
           o1.data_ptr(), o2.data_ptr(), st)
    x = torch.randn((T, d), device=dev).bfloat16()
    w = torch.ones(d, device=dev)
    rstd = torch.ones(T, device=dev)
    invs = [torch.randperm(d, device=dev).int() for _ in range(3)]
    dus = [torch.randn_like(x) for _ in range(3)]
    dx = torch.empty_like(x)
    dw = torch.empty_like(w)
    ws, wsb = N.workspace(N.lib().poetx_rmsnorm_gather_bwd_workspace_bytes(T, d))
    N.call("poetx_rmsnorm_gather_bwd", T, d, x.data_ptr(), w.data_ptr(), rstd.data_ptr(), 3, _ptrs(invs), _ptrs(dus),
           None, dx.data_ptr(), dw.data_ptr(), 0, ws, wsb, st)
    fwds = [torch.argsort(i.long()).int() for i in invs]
    outs = [torch.empty_like(x) for _ in range(3)]
    N.call("poetx_rmsnorm_gather", T, d, x.data_ptr(), w.data_ptr(), 1e-6, 3, _ptrs(fwds), _ptrs(outs), rstd.data_ptr(), st)
    S_, H_, hd_ = 256, 32, 64
    ang = torch.outer(torch.arange(S_, device=dev).float(), 1.0 / (10000 ** (torch.arange(0, hd_, 2, device=dev).float() / hd_)))
    cs, sn = ang.cos().contiguous(), ang.sin().contiguous()
    ro = torch.empty_like(x)
    N.call("poetx_rope_scatter", T, S_, H_, hd_, x.data_ptr(), invs[0].data_ptr(), cs.data_ptr(), sn.data_ptr(),
           ro.data_ptr(), st)
    from paper_2603_05500_b200.trainer import _Attention
    q_, k_, v_ = (torch.randn((T, d), device=dev).bfloat16().requires_grad_(True) for _ in range(3))
    o_ = _Attention.apply(q_, k_, v_, T // S_, S_, H_, hd_)
    torch.autograd.grad(o_, (q_, k_, v_), torch.randn_like(o_))
    torch.cuda.synchronize()


def _long_csv_to_wide(path):
    """`ncu --csv --metrics ... --log-file x.csv` (one row per metric) ->
    the raw page's layout: header, units, one row per kernel launch."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ni, ui, vi, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    launches, units = {}, {}
    for r in rows[1:]:
        e = launches.setdefault(r[ii], {"Kernel Name": r[ki]})
        e[r[ni]] = r[vi].replace(",", "")
        units[r[ni]] = r[ui]
    names = ["Kernel Name"] + sorted(units)
    data = [[launches[k].get(n, "0") for n in names] for k in sorted(launches, key=int)]
    return names, [""] + [units[n] for n in names[1:]], data


def summary(rep):
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        peaks = json.load(fh)
    hbm, tf = peaks["hbm_gbs"], peaks["bf16_tflops"]
    if rep.endswith(".csv"):
        h, units, data = _long_csv_to_wide(rep)
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                              "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,"
                              "dram__throughput.avg.pct_of_peak_sustained_elapsed"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, units, data = rows[0], rows[1], rows[2:]
    col = {k: h.index(k) for k in h}
    scale = {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}
    byte_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    print("| kernel | ncu time | achieved | of peak | ncu DRAM bytes | tensor pipe |")
    print("|---|---|---|---|---|---|")
    i = 0
    for sub, label, kind, work in PLAN:
        j = i
        while j < len(data) and sub not in data[j][col["Kernel Name"]]:
            j += 1
        if j >= len(data):  # not launched at this shape (e.g. no split-T reduce): skip the row
            continue
        r = data[j]
        i = j + 1
        tsec = float(r[col["gpu__time_duration.sum"]]) * scale.get(units[col["gpu__time_duration.sum"]], 1e-6)
        rd = float(r[col["dram__bytes_read.sum"]]) * byte_scale.get(units[col["dram__bytes_read.sum"]], 1)
        wr = float(r[col["dram__bytes_write.sum"]]) * byte_scale.get(units[col["dram__bytes_write.sum"]], 1)
        tp = r[col["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]] or "0"
        if kind == "flop":
            ach = work / tsec / 1e12
            txt, frac = f"{ach:.0f} TFLOP/s", ach / tf
        else:
            ach = work / tsec / 1e9
            txt, frac = f"{ach:.0f} GB/s", ach / hbm
        print(f"| {label} | {tsec * 1e6:.1f} us | {txt} | {frac:.2f} | {(rd + wr) / 1e6:.1f} MB | {float(tp):.0f}% |")
    print(f"\nPeaks: MEASURED_PEAKS.json burst figures (kernels timed alone): {hbm} GB/s HBM, {tf} TFLOP/s bf16.")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summary":
        summary(sys.argv[2])
    else:
        run()
