// tcgen05 / TMEM / TMA tensor-core kernels for the BF16 path (sm_100a).
// Each entry returns POETX_ENOTSUPPORTED when a shape does not tile, and
// the caller falls back to the SIMT kernel.
#pragma once

#include "common.cuh"
#include "simt_gemm.cuh"

namespace poetx {

constexpr int POETX_ENOTSUPPORTED = -100;  // internal: "use another kernel"

bool tc_enabled();

// C[M,N] = op(A) op(B), BF16 in, fp32 accumulate (TMEM), BF16 out.
int tc_matmul(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA,
              const void* B, int64_t ldb, int transB, void* C, int64_t ldc, cudaStream_t st);

// y_s = x_s g[s] (or g[s]^T) for every length-b segment s; BF16.
int tc_blockdiag(const GemmDesc& d, cudaStream_t st);

// out[s] = sum_t x_s^T y_s, BF16 in, fp32 out (overwrites out).
size_t tc_outer_ws_bytes(int64_t T, int64_t nb, int64_t b);
int tc_segmented_outer(int64_t T, int64_t nb, int64_t b, const void* x, const void* y, float* out,
                       Workspace& ws, cudaStream_t st);

}  // namespace poetx
