"""Kernel microbenchmarks on one GPU (CUDA-event timing, warm L2 noted).

    python tools/microbench.py [gemm|layer|all]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2603_05500_b200 import _native as N


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def gemm():
    print("== tcgen05 GEMM vs cuBLAS (bf16) ==")
    for M, Nn, K in [(8192, 2048, 2048), (8192, 5632, 2048), (8192, 2048, 5632), (16384, 4096, 4096)]:
        for tb in (0, 1):
            a = torch.randn((M, K), device="cuda").bfloat16()
            b = torch.randn((Nn, K) if tb else (K, Nn), device="cuda").bfloat16()
            c = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)

            def ours():
                N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, b.data_ptr(), b.shape[1], tb,
                       c.data_ptr(), Nn, 0, N.stream_ptr())
            ms = timeit(ours)
            bt = b.t() if tb else b
            ms_cublas = timeit(lambda: torch.matmul(a, bt))
            fl = 2.0 * M * Nn * K
            print(f"M={M} N={Nn} K={K} transB={tb}: ours {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s | "
                  f"cuBLAS {ms_cublas:.3f} ms {fl / ms_cublas / 1e9:.0f} TF/s")


def layer():
    import paper_2603_05500_b200 as P
    from paper_2603_05500_b200.trainer import PoetLinear, PoetStack
    print("== POET-X layer (bf16, b=256, T=8192) ==")
    T = 8192
    for m, n in [(2048, 2048), (2048, 5632), (5632, 2048)]:
        b = 256
        st = PoetStack([("x.r", m // b), ("x.p", n // b)], b, torch.device("cuda"))
        lay = PoetLinear("x", m, n, st, P.Rng(0))
        x = torch.randn((T, m), device="cuda").bfloat16().requires_grad_(True)
        dz = torch.randn((T, n), device="cuda").bfloat16()

        def fwd():
            return lay(x)

        def fwdbwd():
            z = lay(x)
            z.backward(dz)
        t_cf = timeit(st.forward_factors, 5, 1)
        t_cb = timeit(st.backward_factors, 5, 1)
        t_fw = timeit(fwd, 5, 1)
        t_fb = timeit(fwdbwd, 5, 1)
        gemm_ms = 2 * 2.0 * T * m * n / 1.4e15 * 1e3
        print(f"{m}->{n}: cnp fwd {t_cf:.3f} ms, cnp bwd {t_cb:.3f} ms, layer fwd {t_fw:.3f} ms, "
              f"fwd+bwd {t_fb:.3f} ms (2 GEMMs at 1.4 PF would be {gemm_ms:.3f} ms)")
    print("== model-batched CNP, Llama-1B (3696 blocks of 256) ==")
    nb, b = 3696, 256
    st = PoetStack([("all", nb)], b, torch.device("cuda"))
    st.group.param.normal_(0, 0.01)
    t_cf = timeit(st.forward_factors, 5, 1)
    t_cb = timeit(st.backward_factors, 5, 1)
    fl_f, fl_b = 2 * 3 * nb * b ** 3, 2 * 4 * nb * b ** 3
    print(f"cnp fwd {t_cf:.3f} ms ({fl_f / t_cf / 1e9:.0f} TF/s), cnp bwd {t_cb:.3f} ms ({fl_b / t_cb / 1e9:.0f} TF/s)")


def hbm():
    import paper_2603_05500_b200 as P
    print("== HBM-bound kernels (bf16, T=8192) ==")
    T = 8192
    for cols in (2048, 5632):
        x = torch.randn((T, cols), device="cuda").bfloat16()
        pm = P.sample_permutation(cols, P.Rng(1))
        ms = timeit(lambda: P.permute_features(x, pm, "inverse"))
        print(f"permute T x {cols}: {ms * 1e3:.1f} us  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
        for b in (256, 64):
            G = P.BlockDiagonalFactor((0.1 * torch.randn((cols // b, b, b), device="cuda")).bfloat16())
            for tr in (False, True):
                ms = timeit(lambda: P.apply_to_features(G, x, transpose=tr))
                print(f"apply b={b} T x {cols} transpose={tr}: {ms * 1e3:.1f} us  "
                      f"{2 * x.numel() * 2 / ms / 1e6:.0f} GB/s  {2 * x.numel() * b / ms / 1e9:.0f} TF/s")
            y = torch.randn_like(x)
            ms = timeit(lambda: P.segmented_outer(x, y, b))
            print(f"segmented_outer b={b} T x {cols}: {ms * 1e3:.1f} us  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s "
                  f"{2 * x.numel() * b / ms / 1e9:.0f} TF/s")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("gemm", "all"):
        gemm()
    if what in ("hbm", "all"):
        hbm()
    if what in ("layer", "all"):
        layer()
