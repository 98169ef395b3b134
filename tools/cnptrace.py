"""Phase timeline of the fused CNP kernels (build-time probe).

    bash tools/variant_build.sh ctrace -DPOETX_CNP_TRACE
    POETX_LIB_PATH=abtest/lib_ctrace.so python tools/cnptrace.py [nb] [b]

Thread 0 of every CTA stamps globaltimer at each phase boundary of its
first five blocks; printed: mean / max phase durations over CTAs (blocks
1-4; block 0 includes the launch ramp) and the per-block total."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_05500_b200 import _native as N

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 3696
b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
lib = N.lib()
pairs = b * (b - 1) // 2
packed = (0.02 * torch.randn((nb, pairs), device="cuda")).contiguous()
dg = torch.randn((nb, b, b), device="cuda")
g16 = torch.empty((nb, b, b), device="cuda", dtype=torch.bfloat16)
dp = torch.empty((nb, pairs), device="cuda")
FWD = ["start", "unpack 2Q", "MMA (2Q)^2", "S1,S0 <- Q^2, Q^2-2Q", "MMA Q^2 H", "G epilogue", "G store + sync"]
BWD = ["start", "unpack Q", "dG tiles E,F (+A1<-E)", "MMA QE, FQ, QF", "S2<-QE, S1<-Z", "MMA QQ, (QE)Q",
       "S0 <- Q^2", "MMA ZQ^2, Q^2Z", "stage A1 (fp32)", "packed output + sync"]


def run(fwd):
    if fwd:
        N.call("poetx_cnp_forward_fused", nb, b, packed.data_ptr(), g16.data_ptr(), None, N.stream_ptr())
    else:
        N.call("poetx_cnp_backward_fused", nb, b, packed.data_ptr(), dg.data_ptr(), dp.data_ptr(), 0, N.stream_ptr())


for fwd, names in ((True, FWD), (False, BWD)):
    for _ in range(3):
        run(fwd)
    torch.cuda.synchronize()
    lib.poetx_cnp_trace_reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(fwd)
    e1.record()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (512 * 64))()
    lib.poetx_cnp_trace_copy(buf, 512 * 64)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(512, 64).astype(np.int64)
    ctas = [i for i in range(512) if t[i, 0] > 0]
    if hasattr(lib, "poetx_cnp_trace_copy_w"):
        bw = (C.c_ulonglong * (512 * 32))()
        lib.poetx_cnp_trace_copy_w(bw, 512 * 32)
        tw = np.frombuffer(bw, dtype=np.uint64).reshape(512, 32).astype(np.int64)
        for rk in ((0, 1) if b == 256 else (0,)):
            sub = [i for i in ctas if (i % 2 == rk or b != 256) and tw[i, 0] > 0]
            if sub:
                per = [np.mean([(tw[i, 2 * w + 1] - tw[i, 2 * w]) / 1000.0 for i in sub]) for w in range(8)]
                print(f"   rank {rk} per-warp scatter (block 1): " + " ".join(f"{x:.2f}" for x in per))
                if not fwd and all(tw[i, 16] > 0 for i in sub):
                    per = [np.mean([(tw[i, 17 + 2 * w] - tw[i, 16 + 2 * w]) / 1000.0 for i in sub]) for w in range(8)]
                    print(f"   rank {rk} per-warp output (block 1): " + " ".join(f"{x:.2f}" for x in per))
    nph = len(names)
    for rk in ((0, 1) if b == 256 else (0,)):
        sub = [i for i in ctas if i % 2 == rk] if b == 256 else ctas
        w, sc = [], []
        for i in sub:
            for it in range(1, 5):
                t0, tw, t1 = t[i, it * 12], t[i, it * 12 + 10], t[i, it * 12 + 11]
                if t0 > 0 and tw > 0 and t1 > 0:
                    w.append((tw - t0) / 1000.0)
                    sc.append((t1 - tw) / 1000.0)
        if w:
            print(f"   rank {rk}: staging wait {np.mean(w):.2f} us, scatter part 1 {np.mean(sc):.2f} us")
    d = []  # [cta, block, phase] durations
    for i in ctas:
        for it in range(1, 5):
            row = t[i, it * 12: it * 12 + nph]
            if (row > 0).all():
                d.append(np.diff(row) / 1000.0)
    d = np.array(d)
    blk = d.sum(axis=1)
    if b == 256:
        for rk in (0, 1):
            dd = []
            for i in ctas:
                if i % 2 != rk:
                    continue
                for it in range(1, 5):
                    row = t[i, it * 12: it * 12 + nph]
                    if (row > 0).all():
                        dd.append(np.diff(row) / 1000.0)
            dd = np.array(dd)
            print(f"   rank {rk} phases: " + "  ".join(f"{x:.2f}" for x in dd.mean(axis=0)))
    print(f"== {'forward' if fwd else 'backward'} b={b}, {nb} blocks, {len(ctas)} CTAs: launch {e0.elapsed_time(e1) * 1000:.1f} us, "
          f"{e0.elapsed_time(e1) * 1000 / max(1, nb / (len(ctas) // (2 if b == 256 else 1))):.2f} us per block round")
    print(f"   per block (thread 0, blocks 1-4): mean {blk.mean():.2f} us  (min {blk.min():.2f}, max {blk.max():.2f})")
    for k in range(nph - 1):
        print(f"   {names[k + 1]:28s} mean {d[:, k].mean():6.2f} us  max {d[:, k].max():6.2f}  ({100 * d[:, k].mean() / blk.mean():4.1f}%)")
    # next block start - this block end
    gaps = [(t[i, (it + 1) * 12] - t[i, it * 12 + nph - 1]) / 1000.0 for i in ctas for it in range(1, 4)
            if t[i, (it + 1) * 12] > 0 and t[i, it * 12 + nph - 1] > 0]
    if gaps:
        print(f"   end -> next block start mean {np.mean(gaps):.2f} us")
