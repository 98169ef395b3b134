"""POET-XQ GEMM timing: the fused int8 pair GEMM (poetx_matmul_q8) against
dequantize + bf16 GEMM and the plain bf16 GEMM, Llama-8B (T = 1024) and
Llama-1B (T = 8192) projection shapes.  CUDA events, mean of 20."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_05500_b200 import _native as N


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / iters


print("== POET-XQ GEMM: fused int8 producer vs dequantize + GEMM ==")
for M, Nn, K in [(1024, 4096, 4096), (1024, 14336, 4096), (1024, 4096, 14336), (8192, 2048, 2048), (8192, 5632, 2048)]:
    for tb in (0, 1):
        a = torch.randn((M, K), device="cuda").bfloat16()
        rows, cols = (Nn, K) if tb else (K, Nn)
        codes = torch.randint(-127, 128, (rows, cols), device="cuda", dtype=torch.int8)
        sc = torch.rand(rows, device="cuda") * 0.01
        w = torch.empty((rows, cols), device="cuda", dtype=torch.bfloat16)
        c = torch.empty((M, Nn), device="cuda", dtype=torch.bfloat16)
        st = N.stream_ptr()
        q8 = timeit(lambda: N.call("poetx_matmul_q8", M, Nn, K, a.data_ptr(), K, codes.data_ptr(), cols, tb,
                                   sc.data_ptr(), c.data_ptr(), Nn, st))

        def deq():
            N.call("poetx_dequantize_rows", N.BF16, rows, cols, cols, codes.data_ptr(), sc.data_ptr(), None, None,
                   w.data_ptr(), st)
            N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, w.data_ptr(), cols, tb, c.data_ptr(), Nn, 0, st)
        dq = timeit(deq)
        bf = timeit(lambda: N.call("poetx_matmul", N.BF16, M, Nn, K, a.data_ptr(), K, 0, w.data_ptr(), cols, tb,
                                   c.data_ptr(), Nn, 0, st))
        fl = 2.0 * M * Nn * K
        print(f"M={M} N={Nn} K={K} transB={tb}: q8 {q8:.3f} ms ({fl / q8 / 1e9:.0f} TF/s) | dequant+gemm {dq:.3f} ms | "
              f"bf16 gemm alone {bf:.3f} ms ({fl / bf / 1e9:.0f} TF/s)")
