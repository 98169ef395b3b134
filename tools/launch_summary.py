"""Family shares of an ncu launch list (gpu__time_duration.sum per launch,
--csv --log-file): python tools/launch_summary.py launches.csv"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
FAMILIES = [
    ("tc2_kernel", "tcgen05 CTA-pair GEMM (mm2/adjoint/outer/CNP/folds)"), ("tc_kernel", "tcgen05 single-CTA GEMM"),
    ("bd_kernel", "block-diagonal apply"), ("reduce_splits", "split-T reduce"), ("rmsnorm", "rmsnorm+gather"),
    ("colsum", "rmsnorm+gather"), ("swiglu", "swiglu+gather"), ("rope", "rope+scatter"),
    ("scatter_add", "residual scatter"), ("permute", "permute"), ("unpack_q", "CNP glue"), ("combine_fwd", "CNP glue"),
    ("bwd_prep", "CNP glue"), ("pack_dq", "CNP glue"), ("to_bf16", "CNP glue"), ("adamw", "AdamW+norm"),
    ("sqdev", "AdamW+norm"), ("sdpa", "attention"), ("cudnn", "attention"), ("attn_bwd", "attention"),
    ("nvjet", "lm_head GEMMs (cuBLAS)"), ("ce_fwd", "cross-entropy"), ("ce_bwd", "cross-entropy"),
    ("dequant", "POET-XQ"), ("quant", "POET-XQ"), ("cnp_fused", "CNP fused (tcgen05)"), ("merge_tc", "merge (tcgen05)"),
]


def family(name):
    for k, f in FAMILIES:
        if k in name:
            return f
    return "other"


rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
fam = collections.defaultdict(lambda: [0.0, 0])
for r in rows[1:]:
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    f = fam[family(r[ki])]
    f[0] += us
    f[1] += 1
tot = sum(v[0] for v in fam.values())
print(f"{len(rows) - 1} launches, {tot / 1e3:.2f} ms of serialised kernel time")
print("| family | ms | share | launches |\n|---|---|---|---|")
for k, (us, n) in sorted(fam.items(), key=lambda x: -x[1][0]):
    print(f"| {k} | {us / 1e3:.2f} | {100 * us / tot:.1f}% | {n} |")
