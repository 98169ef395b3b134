"""Merge product timing at Llama shapes: the tensor-core K9 kernel
(poetx_merge_tc) vs the CUDA-core fp32 passes it replaces, and one whole
Llama-1B layer set (7 projections).  CUDA events, best of 5.

    python tools/mergebench.py [m n]     (one shape, for ncu)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N


def best(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    out = 1e9
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        e.synchronize()
        out = min(out, a.elapsed_time(e))
    return out


def shape(m, n, b=256, reps=5):
    g_r = torch.eye(b, device="cuda").expand(m // b, b, b).contiguous() + 0.01 * torch.randn((m // b, b, b), device="cuda")
    g_p = torch.eye(b, device="cuda").expand(n // b, b, b).contiguous() + 0.01 * torch.randn((n // b, b, b), device="cuda")
    pm = torch.randn((m, n), device="cuda").to(torch.bfloat16)
    out = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    st = N.stream_ptr()
    tc = best(lambda: N.call("poetx_merge_tc", m, n, b, g_r.data_ptr(), g_p.data_ptr(), pm.data_ptr(), None, None, n,
                             out.data_ptr(), N.BF16, n, st), reps)
    # the CUDA-core path it replaces: bf16 -> fp32, two fp32 block-diagonal passes
    pm32, mid1, mid2 = (torch.empty((m, n), device="cuda") for _ in range(3))

    def simt():
        pm32.copy_(pm)
        N.call("poetx_apply_to_weight_rows", N.F32, m // b, b, n, g_r.data_ptr(), 0, pm32.data_ptr(),
               mid1.data_ptr(), st)
        N.call("poetx_apply_to_features", N.F32, m, n // b, b, g_p.data_ptr(), 0, mid1.data_ptr(), mid2.data_ptr(), st)
    try:
        cc = best(simt, 2)
    except Exception as e:  # noqa: BLE001
        cc = float("nan")
        print("simt path:", e)
    fl = 5 * 2.0 * b ** 3 * (m // b) * (n // b)
    byt = m * n * 2 * 2 + (m + n) * b * 4
    return tc, cc, fl, byt


if __name__ == "__main__":
    if len(sys.argv) > 2:
        shape(int(sys.argv[1]), int(sys.argv[2]), reps=2)
        sys.exit(0)
    print("== K9 tensor-core merge product (bf16x3 split, b=256) vs CUDA-core fp32 passes ==")
    tot_tc = tot_cc = 0.0
    for m, n, cnt in [(2048, 2048, 4), (2048, 5632, 2), (5632, 2048, 1)]:
        tc, cc, fl, byt = shape(m, n)
        tot_tc += cnt * tc
        tot_cc += cnt * cc
        print(f"{m}x{n}: tc {tc:.3f} ms ({fl / tc / 1e9:.0f} TF/s on 5 products, {byt / tc / 1e6:.0f} GB/s of "
              f"PM+out+factors) | cuda-core {cc:.3f} ms | x{cc / tc:.1f}")
    print(f"one Llama-1B decoder block (7 projections): tc {tot_tc:.2f} ms, cuda-core {tot_cc:.2f} ms; "
          f"x24 layers: {24 * tot_tc:.1f} vs {24 * tot_cc:.1f} ms")
