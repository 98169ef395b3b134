// tcgen05 / TMEM / TMA tensor-core kernels for the BF16 path (sm_100a).
// Each entry returns POETX_ENOTSUPPORTED when a shape does not tile, and
// the caller falls back to the SIMT kernel.
#pragma once

#include "common.cuh"
#include "simt_gemm.cuh"

namespace poetx {

constexpr int POETX_ENOTSUPPORTED = -100;  // internal: "use another kernel"

bool tc_enabled();

// A bf16 operand: row-major [rows, cols] view with a row pitch (elements).
// K-major: the contraction index runs along cols; MN-major: along rows.
struct TcOperand {
  const void* ptr;
  int64_t rows, cols, pitch;
  bool mn_major;
  // POET-XQ B operand: int8 codes (pitch in bytes = elements) whose ROW r of
  // this [rows, cols] view carries the fp32 scale row_scale[r]; converted to
  // bf16 (code * scale, one rounding, as the dequantizer) on chip
  const float* row_scale = nullptr;
};

// Grouped/split-K problem: for g < groups, s < splits,
//   C[g*c_goff + s*c_soff + m*ldc + n] = alpha * sum_{k in split s} A_g[m,k] B_g[k,n]
// where group g shifts the operand TMA coordinates (col, row) by
// (a_g0*g, a_g1*g) and (b_g0*g, b_g1*g).  BF16 or FP32 output.
struct TcProblem {
  int64_t M, N, K;
  int groups, splits, bn;
  int a_g0, a_g1, b_g0, b_g1;
  void* C;
  int64_t ldc, c_goff, c_soff;
  int out_f32;
  int accumulate;  // fp32 output only: C += alpha * AB
  float alpha;
  const char* name;
  int ms;  // 2: two 128-row M sub-tiles per CTA share each B stage (A and B MN-major)
  int tma_epi;  // 1: stage the epilogue in smem and write C with TMA bulk stores
};

int tc_grouped(const TcOperand& A, const TcOperand& B, const TcProblem& p, cudaStream_t st);

// C[M,N] = op(A) op(B), BF16 in, fp32 accumulate (TMEM), BF16 out.
int tc_matmul(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA,
              const void* B, int64_t ldb, int transB, void* C, int64_t ldc, cudaStream_t st);
// same with B = int8 codes [K, N] (transB = 0: row k scaled by scales[k]) or
// [N, K] (transB = 1: row n scaled by scales[n]), i.e. the POET-XQ premerged
// weight dequantized inside the GEMM producer; ENOTSUPPORTED off the pair path
int tc_matmul_q8(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA,
                 const int8_t* B, int64_t ldb, int transB, const float* scales, void* C, int64_t ldc,
                 cudaStream_t st);

// y_s = x_s g[s] (or g[s]^T) for every length-b segment s; BF16.
int tc_blockdiag(const GemmDesc& d, cudaStream_t st);
int tc_blockdiag_apply(int64_t T, int64_t nb, int64_t b, const void* g, int transpose,
                       const void* x, void* y, cudaStream_t st);

// split-K factor used by the tensor-core segmented outer product
int tc_outer_splits(int64_t T, int64_t nb, int64_t b);
size_t tc_outer_ws_bytes(int64_t T, int64_t nb, int64_t b);

}  // namespace poetx
