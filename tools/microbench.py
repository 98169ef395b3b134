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
            N.lib().poetx_set_gemm_pair_ms(2)
            ms = timeit(ours)
            ref = torch.matmul(a.float(), (b.t() if tb else b).float())
            err2 = float((c.float() - ref).abs().max() / ref.abs().max())
            N.lib().poetx_set_gemm_pair_ms(1)
            ms_p1 = timeit(ours)
            N.lib().poetx_set_gemm_pair_ms(0)
            N.lib().poetx_set_gemm_pair_enabled(0)
            ms1 = timeit(ours)
            N.lib().poetx_set_gemm_pair_enabled(1)
            bt = b.t() if tb else b
            ms_cublas = timeit(lambda: torch.matmul(a, bt))
            fl = 2.0 * M * Nn * K
            print(f"M={M} N={Nn} K={K} transB={tb}: ours(pair 512x256) {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s "
                  f"(rel err {err2:.1e}) | pair 256x256 {fl / ms_p1 / 1e9:.0f} TF/s | 1cta {fl / ms1 / 1e9:.0f} TF/s | "
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
        print(f"permute T x {cols}: {ms * 1e3:.1f} us  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s "
              f"(env POETX_PERMUTE_T8={os.environ.get('POETX_PERMUTE_T8', '1')})")
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


def rows():
    import ctypes as C
    from paper_2603_05500_b200.trainer import _ptrs
    print("== fused row kernels (bf16, T=8192) ==", os.environ.get("POETX_ROW_TILE_KB", "48"), "KB tiles")
    T, d, f, H, hd, S = 8192, 2048, 5632, 32, 64, 256
    dev = "cuda"
    st = N.stream_ptr()
    x = torch.randn((T, d), device=dev).bfloat16()
    w = torch.ones(d, device=dev)
    perms = [torch.randperm(d, device=dev).int() for _ in range(3)]
    outs = [torch.empty_like(x) for _ in range(3)]
    rstd = torch.empty(T, device=dev)
    ms = timeit(lambda: N.call("poetx_rmsnorm_gather", T, d, x.data_ptr(), w.data_ptr(), 1e-6, 3, _ptrs(perms),
                               _ptrs(outs), rstd.data_ptr(), st))
    print(f"rmsnorm_gather K=3: {ms * 1e3:.1f} us  {4 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
    dx = torch.empty_like(x)
    dw = torch.empty_like(w)
    ws, wsb = N.workspace(N.lib().poetx_rmsnorm_gather_bwd_workspace_bytes(T, d))
    ms = timeit(lambda: N.call("poetx_rmsnorm_gather_bwd", T, d, x.data_ptr(), w.data_ptr(), rstd.data_ptr(), 3,
                               _ptrs(perms), _ptrs(outs), outs[1].data_ptr(), dx.data_ptr(), dw.data_ptr(), 0,
                               ws, wsb, st))
    print(f"rmsnorm_gather_bwd K=3 (+dres): {ms * 1e3:.1f} us  {6 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
    vg = torch.randn((T, f), device=dev).bfloat16()
    vu = torch.randn_like(vg)
    o = torch.empty_like(vg)
    pf = [torch.randperm(f, device=dev).int() for _ in range(4)]
    ms = timeit(lambda: N.call("poetx_swiglu_gather", T, f, vg.data_ptr(), vu.data_ptr(), pf[0].data_ptr(),
                               pf[1].data_ptr(), o.data_ptr(), st))
    print(f"swiglu_gather: {ms * 1e3:.1f} us  {3 * vg.numel() * 2 / ms / 1e6:.0f} GB/s")
    o2 = torch.empty_like(vg)
    ms = timeit(lambda: N.call("poetx_swiglu_gather_bwd", T, f, vg.data_ptr(), vu.data_ptr(), o.data_ptr(),
                               pf[0].data_ptr(), pf[1].data_ptr(), pf[2].data_ptr(), pf[3].data_ptr(),
                               o2.data_ptr(), outs[0].data_ptr() if False else torch.empty_like(vg).data_ptr(), st))
    print(f"swiglu_gather_bwd: {ms * 1e3:.1f} us  {5 * vg.numel() * 2 / ms / 1e6:.0f} GB/s")
    ang = torch.outer(torch.arange(S, device=dev).float(), torch.rand(hd // 2, device=dev))
    cs, sn = ang.cos().contiguous(), ang.sin().contiguous()
    ms = timeit(lambda: N.call("poetx_rope_scatter", T, S, H, hd, x.data_ptr(), perms[0].data_ptr(), cs.data_ptr(),
                               sn.data_ptr(), outs[1].data_ptr(), st))
    print(f"rope_scatter: {ms * 1e3:.1f} us  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
    ms = timeit(lambda: N.call("poetx_rope_scatter_bwd", T, S, H, hd, x.data_ptr(), perms[0].data_ptr(),
                               cs.data_ptr(), sn.data_ptr(), outs[1].data_ptr(), st))
    print(f"rope_scatter_bwd: {ms * 1e3:.1f} us  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s")
    ms = timeit(lambda: N.call("poetx_scatter_add", T, d, x.data_ptr(), outs[0].data_ptr(), perms[0].data_ptr(),
                               outs[2].data_ptr(), st))
    print(f"scatter_add: {ms * 1e3:.1f} us  {3 * x.numel() * 2 / ms / 1e6:.0f} GB/s")


def cnp():
    from paper_2603_05500_b200.trainer import PoetStack
    print("== model-batched CNP, Llama-1B (3696 blocks of 256) ==")
    nb, b = 3696, 256
    st = PoetStack([("all", nb)], b, torch.device("cuda"))
    st.group.param.normal_(0, 0.01)
    t_cf = timeit(st.forward_factors, 5, 1)
    t_cb = timeit(st.backward_factors, 5, 1)
    fl_f, fl_b = 2 * 3 * nb * b ** 3, 2 * 4 * nb * b ** 3
    print(f"cnp fwd {t_cf:.3f} ms ({fl_f / t_cf / 1e9:.0f} TF/s), cnp bwd {t_cb:.3f} ms ({fl_b / t_cb / 1e9:.0f} TF/s)")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("gemm", "all"):
        gemm()
    if what in ("rows", "all"):
        rows()
    if what in ("hbm", "all"):
        hbm()
    if what == "cnp":
        cnp()
    if what in ("layer", "all"):
        layer()
