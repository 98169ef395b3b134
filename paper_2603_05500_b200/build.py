"""Build the in-tree CUDA library libpoetx_b200.so for sm_100a with nvcc.

    python -m paper_2603_05500_b200.build      (or __graft_entry__.build())

The shared object lands next to this file so it travels to the GPU box
with the repo snapshot; the CUDA runtime is linked statically.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpoetx_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["ops.cu", "layer.cu", "tc_gemm.cu", "tc_blockdiag.cu", "cnp_tc.cu", "cnp_fused.cu", "merge_tc.cu", "model_ops.cu", "quant.cu", "attention.cu", "svd.cu", "prof.cu", "philox.cpp"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    "-shared", "-cudart", "static",
]


def _deps():
    deps = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC))
    deps.append(os.path.join(HERE, "..", "include", "poetx_b200.h"))
    deps.append(__file__)
    return [p for p in deps if os.path.isfile(p)]


def source_hash() -> str:
    """Content hash of every source the library is built from (robust to the
    mtimes a repo snapshot copy may reset)."""
    h = hashlib.sha256()
    for p in _deps():
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".sha"):
        return True
    with open(LIB + ".sha") as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    digest = source_hash()
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    tmp = LIB + ".tmp"
    cmd = [NVCC, *FLAGS, "-o", tmp, *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    with open(LIB + ".sha", "w") as f:
        f.write(digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
