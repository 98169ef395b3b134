"""Per-CTA timeline of one pair-GEMM launch (build-time probe).

    bash tools/variant_build.sh trace -DPOETX_GEMM_TRACE
    POETX_LIB_PATH=abtest/lib_trace.so python tools/gemmtrace.py M N K transB [ms]

Prints, per CTA pair (leader stamps), the setup time, each tile's
first-MMA / last-MMA / epilogue window relative to the earliest kernel
entry, and a summary: where the launch's critical path goes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_05500_b200 import _native as N

M, Nn, K, tb = (int(v) for v in sys.argv[1:5])
ms = int(sys.argv[5]) if len(sys.argv) > 5 else 0
lib = N.lib()
if ms:
    lib.poetx_set_gemm_pair_ms(ms)
a = torch.randn((M, K), device="cuda").bfloat16()
b = torch.randn((Nn, K) if tb else (K, Nn), device="cuda").bfloat16()
c = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)


def run():
    N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, b.data_ptr(), b.shape[1], tb, c.data_ptr(), Nn, 0,
           N.stream_ptr())


for _ in range(5):
    run()
torch.cuda.synchronize()
reps = []
for _ in range(3):
    lib.poetx_gemm_trace_reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (512 * 64))()
    lib.poetx_gemm_trace_copy(buf, 512 * 64)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(512, 64).astype(np.int64)
    reps.append((t, e0.elapsed_time(e1)))
t, ev_ms = reps[-1]
ctas = [i for i in range(512) if t[i, 0] > 0]
t0 = min(t[i, 0] for i in ctas)
rel = lambda v: (v - t0) / 1000.0 if v > 0 else float("nan")  # us
print(f"shape {M}x{Nn}x{K} transB={tb} ms={ms or 'auto'}: {len(ctas)} CTAs, event {ev_ms * 1000:.1f} us, "
      f"last end {max(rel(t[i, 2]) for i in ctas):.1f} us after first entry")
entry = np.array([rel(t[i, 0]) for i in ctas])
setup = np.array([rel(t[i, 1]) - rel(t[i, 0]) for i in ctas])
print(f"entry spread {entry.min():.2f}..{entry.max():.2f} us; setup (init+alloc+cluster sync) mean {setup.mean():.2f} max {setup.max():.2f} us")
rows = []
for i in ctas[::2]:  # leaders
    tiles = []
    for j in range(12):
        s = 4 + j * 5
        if t[i, s + 2] == 0 and t[i, s + 0] == 0:
            break
        tiles.append((rel(t[i, s + 4]), rel(t[i, s + 0]), rel(t[i, s + 1]), rel(t[i, s + 2]), rel(t[i, s + 3])))
    rows.append((i, rel(t[i, 0]), rel(t[i, 1]), tiles, rel(t[i, 2])))
for i, en, su, tiles, end in rows[:12] + rows[-4:]:
    ts = "  ".join(f"[tma {a:.1f} mma {b:.1f}-{c:.1f} epi {d:.1f}-{e:.1f}]" for a, b, c, d, e in tiles)
    print(f"cta {i:3d} entry {en:5.1f} setup {su:5.1f} {ts} end {end:5.1f}")
# summary
first_tma = np.array([r[3][0][0] - r[2] for r in rows if r[3]])
main = np.array([tt[2] - tt[1] for r in rows for tt in r[3]])
epi = np.array([tt[4] - tt[3] for r in rows for tt in r[3]])
tail = np.array([r[4] - r[3][-1][4] for r in rows if r[3]])
ntiles = np.array([len(r[3]) for r in rows])
print(f"tiles per pair {np.bincount(ntiles)}; setup->first TMA {first_tma.mean():.2f} us; first TMA->first MMA "
      f"{np.mean([r[3][0][1] - r[3][0][0] for r in rows if r[3]]):.2f} us")
print(f"mainloop per tile mean {main.mean():.2f} (min {main.min():.2f} max {main.max():.2f}) us; epilogue per tile "
      f"mean {epi.mean():.2f} us; last epi -> end {tail.mean():.2f} us")
rel0 = [(rel(t[i, 60]) - rel(t[i, 6]), rel(t[i, 61]) - rel(t[i, 6])) for i in ctas[::2] if t[i, 60] > 0]
if rel0:
    print(f"tile 0: epilogue start -> sub-tile 0 released {np.mean([a for a, b in rel0]):.2f} us, -> sub-tile 1 released "
          f"{np.mean([b for a, b in rel0]):.2f} us")
gaps = [r[3][j + 1][1] - r[3][j][2] for r in rows for j in range(len(r[3]) - 1)]
if gaps:
    print(f"gap last MMA(j) -> first MMA(j+1) mean {np.mean(gaps):.2f} us")
