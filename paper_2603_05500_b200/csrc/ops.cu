// Elementwise, permutation, block-diagonal, CNP and optimizer entry points
// of the poetx_b200 C ABI (see include/poetx_b200.h for the contract and
// the reference functions each one replaces).
#include <cmath>
#include <type_traits>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "simt_gemm.cuh"
#include "tc_gemm.cuh"
#include "tile8.cuh"

namespace poetx {

// ----------------------------------------------------------------- errors --
static thread_local std::string g_last_error;
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}

// ------------------------------------------------------- GEMM dispatch ----
// GEMM on dtype `dt` operands with output in `out_dt` (BF16 operands may
// write fp32, e.g. segmented_outer partials).
int gemm(int dt, int out_dt, const GemmDesc& d, cudaStream_t st) {
  if (dt == POETX_F32 && out_dt == POETX_F32) return simt_gemm<float, float, float>(d, st);
  if (dt == POETX_F64 && out_dt == POETX_F64) return simt_gemm<double, double, double>(d, st);
  if (dt == POETX_BF16 && out_dt == POETX_BF16)
    return simt_gemm<__nv_bfloat16, __nv_bfloat16, __nv_bfloat16>(d, st);
  if (dt == POETX_BF16 && out_dt == POETX_F32)
    return simt_gemm<__nv_bfloat16, __nv_bfloat16, float>(d, st);
  set_error("gemm: unsupported dtype pair (%d -> %d)", dt, out_dt);
  return POETX_ESHAPE;
}

// Plain (batched) matmul C = op(A) op(B) over contiguous row-major stacks.
static int bmm(int dt, int64_t batch, int64_t M, int64_t N, int64_t K, const void* A, bool tA,
               const void* B, bool tB, void* C, double alpha, double beta, cudaStream_t st) {
  GemmDesc d{};
  d.M = M; d.N = N; d.K = K; d.batch = batch;
  d.A = A; d.sAb = M * K; d.sAm = tA ? 1 : K; d.sAk = tA ? M : 1;
  d.B = B; d.sBb = K * N; d.sBk = tB ? 1 : N; d.sBn = tB ? K : 1;
  d.C = C; d.sCb = M * N; d.sCm = N; d.sCn = 1;
  d.alpha = alpha; d.beta = beta;
  return gemm(dt, dt, d, st);
}

// ------------------------------------------------------- skew packing ----
__device__ __forceinline__ int64_t pair_index(int64_t i, int64_t j, int64_t b) {
  // row-major strict upper triangle (cnp.py:66-68): (0,1),(0,2),...,(1,2),...
  return i * b - i * (i + 1) / 2 + (j - i - 1);
}

template <typename T>
__global__ void skew_unpack_kernel(int64_t nb, int64_t b, const T* __restrict__ packed,
                                   T* __restrict__ q) {
  const int64_t pairs = b * (b - 1) / 2, total = nb * b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e / (b * b), r = e % (b * b), i = r / b, j = r % b;
    T v = T(0);
    if (i < j) v = packed[s * pairs + pair_index(i, j, b)];
    else if (i > j) v = -packed[s * pairs + pair_index(j, i, b)];
    q[e] = v;
  }
}

template <typename T>
__global__ void pack_grad_kernel(int64_t nb, int64_t b, const T* __restrict__ dq,
                                 T* __restrict__ g, int accumulate) {
  const int64_t pairs = b * (b - 1) / 2, total = nb * b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e / (b * b), r = e % (b * b), i = r / b, j = r % b;
    if (i >= j) continue;
    const T* blk = dq + s * b * b;
    T v = blk[i * b + j] - blk[j * b + i];
    T* out = g + s * pairs + pair_index(i, j, b);
    *out = accumulate ? *out + v : v;
  }
}

template <typename T>
static int skew_unpack(int64_t nb, int64_t b, const void* packed, void* q, cudaStream_t st) {
  int64_t total = nb * b * b;
  if (total == 0) return POETX_OK;
  skew_unpack_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(nb, b, static_cast<const T*>(packed),
                                                               static_cast<T*>(q));
  POETX_LAUNCHED("skew_unpack");
  return POETX_OK;
}

template <typename T>
static int pack_grad(int64_t nb, int64_t b, const void* dq, void* g, int acc, cudaStream_t st) {
  int64_t total = nb * b * b;
  if (total == 0 || b < 2) return POETX_OK;
  pack_grad_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(nb, b, static_cast<const T*>(dq),
                                                             static_cast<T*>(g), acc);
  POETX_LAUNCHED("pack_grad");
  return POETX_OK;
}

// ---------------------------------------------------------- CNP (k=3) ----
// G = 2 (Q + Q^2 + Q^3) + Q^4 + I   (cnp.py:109-116, same operation order);
// optional bf16 copy for the tensor-core activation path.
template <typename T>
__global__ void cnp_combine_fwd_kernel(int64_t total, int64_t b, const T* __restrict__ q,
                                       const T* __restrict__ q2, const T* __restrict__ q3,
                                       const T* __restrict__ q4, T* __restrict__ g,
                                       __nv_bfloat16* __restrict__ g16) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    T v = T(2) * ((q[e] + q2[e]) + q3[e]) + q4[e];
    int64_t r = e % (b * b);
    if (r / b == r % b) v = v + T(1);
    g[e] = v;
    if (g16) g16[e] = __float2bfloat16_rn(static_cast<float>(v));
  }
}

// generic k: series = I + sum_i Q^i (cnp.py:117-125)
template <typename T>
__global__ void add_identity_kernel(int64_t total, int64_t b, const T* __restrict__ src,
                                    T* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e % (b * b);
    T v = src ? src[e] : T(0);
    dst[e] = (r / b == r % b) ? v + T(1) : v;
  }
}
template <typename T>
__global__ void accumulate_kernel(int64_t total, const T* __restrict__ src, T* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = dst[e] + src[e];
}
template <typename T>
__global__ void to_bf16_kernel(int64_t total, const T* __restrict__ src, __nv_bfloat16* dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = __float2bfloat16_rn(static_cast<float>(src[e]));
}

// dQ = 2 (N1 + N2) + 2 T3 + T4 + 2 T5 + T6   (cnp.py:143-145, same order)
template <typename T>
__global__ void cnp_combine_bwd_kernel(int64_t total, const T* __restrict__ n1,
                                       const T* __restrict__ n2, const T* __restrict__ t3,
                                       const T* __restrict__ t4, const T* __restrict__ t5,
                                       const T* __restrict__ t6, T* __restrict__ dq) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    T v = T(2) * (n1[e] + n2[e]);
    v = v + T(2) * t3[e];
    v = v + t4[e];
    v = v + T(2) * t5[e];
    v = v + t6[e];
    dq[e] = v;
  }
}

size_t cnp_ws_bytes(int dt, int64_t nb, int64_t b, int k) {
  size_t e = elt_size(dt), blk = static_cast<size_t>(nb * b * b) * e;
  int slots = (k == 3) ? 8 : (k + 6);
  return align_up(blk) * slots + 4096;
}

template <typename T>
static int cnp_forward_t(int dt, int64_t nb, int64_t b, int k, const void* qin, const void* packed,
                         void* g, void* g16, void* q2out, Workspace& ws, cudaStream_t st) {
  const int64_t total = nb * b * b;
  const size_t n = static_cast<size_t>(total);
  T* q = const_cast<T*>(static_cast<const T*>(qin));
  if (!q) {
    q = ws.take<T>(n);
    POETX_REQUIRE(q, POETX_ESHAPE, "cnp_forward: workspace too small");
    POETX_TRY(skew_unpack<T>(nb, b, packed, q, st));
  }
  if (k == 3) {
    T* q2 = q2out ? static_cast<T*>(q2out) : ws.take<T>(n);
    T* q3 = ws.take<T>(n);
    T* q4 = ws.take<T>(n);
    POETX_REQUIRE(q2 && q3 && q4, POETX_ESHAPE, "cnp_forward: workspace too small");
    POETX_TRY(bmm(dt, nb, b, b, b, q, false, q, false, q2, 1.0, 0.0, st));   // Q^2
    POETX_TRY(bmm(dt, nb, b, b, b, q2, false, q, false, q3, 1.0, 0.0, st));  // Q^2 Q
    POETX_TRY(bmm(dt, nb, b, b, b, q2, false, q2, false, q4, 1.0, 0.0, st)); // Q^2 Q^2
    cnp_combine_fwd_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(
        total, b, q, q2, q3, q4, static_cast<T*>(g), static_cast<__nv_bfloat16*>(g16));
    POETX_LAUNCHED("cnp_combine_fwd");
    return POETX_OK;
  }
  // generic k: powers, series, G = (I + Q) series
  T* series = ws.take<T>(n);
  T* ipq = ws.take<T>(n);
  T* prev = ws.take<T>(n);
  T* cur = ws.take<T>(n);
  POETX_REQUIRE(series && ipq && prev && cur, POETX_ESHAPE, "cnp_forward: workspace too small");
  add_identity_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, b, q, series);  // I + Q
  POETX_LAUNCHED("add_identity");
  add_identity_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, b, q, ipq);
  POETX_LAUNCHED("add_identity");
  const T* p = q;
  for (int i = 1; i < k; ++i) {
    POETX_TRY(bmm(dt, nb, b, b, b, p, false, q, false, cur, 1.0, 0.0, st));
    accumulate_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, cur, series);
    POETX_LAUNCHED("accumulate");
    T* t = prev; prev = cur; cur = t; p = prev;
  }
  POETX_TRY(bmm(dt, nb, b, b, b, ipq, false, series, false, g, 1.0, 0.0, st));
  if (g16) {
    to_bf16_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, static_cast<T*>(g),
                                                             static_cast<__nv_bfloat16*>(g16));
    POETX_LAUNCHED("to_bf16");
  }
  return POETX_OK;
}

template <typename T>
static int cnp_backward_t(int dt, int64_t nb, int64_t b, int k, const void* qin,
                          const void* packed, const void* q2in, const void* dgin, void* dqout,
                          void* dpacked, int accumulate, Workspace& ws, cudaStream_t st) {
  const int64_t total = nb * b * b;
  const size_t n = static_cast<size_t>(total);
  const T* dg = static_cast<const T*>(dgin);
  T* q = const_cast<T*>(static_cast<const T*>(qin));
  if (!q) {
    q = ws.take<T>(n);
    POETX_REQUIRE(q, POETX_ESHAPE, "cnp_backward: workspace too small");
    POETX_TRY(skew_unpack<T>(nb, b, packed, q, st));
  }
  T* dq = dqout ? static_cast<T*>(dqout) : ws.take<T>(n);
  POETX_REQUIRE(dq, POETX_ESHAPE, "cnp_backward: workspace too small");
  if (k == 3) {
    const T* q2 = static_cast<const T*>(q2in);
    if (!q2) {
      T* t = ws.take<T>(n);
      POETX_REQUIRE(t, POETX_ESHAPE, "cnp_backward: workspace too small");
      POETX_TRY(bmm(dt, nb, b, b, b, q, false, q, false, t, 1.0, 0.0, st));
      q2 = t;
    }
    T* n2 = ws.take<T>(n);
    T* t3 = ws.take<T>(n);
    T* t4 = ws.take<T>(n);
    T* t5 = ws.take<T>(n);
    T* t6 = ws.take<T>(n);
    POETX_REQUIRE(n2 && t3 && t4 && t5 && t6, POETX_ESHAPE, "cnp_backward: workspace too small");
    // N2 = N1 Q^T + Q^T N1 ; T3 = Q^T N2 ; T4 = (Q^2)^T N2 ; T5 = N1 (Q^2)^T ; T6 = N2 (Q^2)^T
    POETX_TRY(bmm(dt, nb, b, b, b, dg, false, q, true, n2, 1.0, 0.0, st));
    POETX_TRY(bmm(dt, nb, b, b, b, q, true, dg, false, n2, 1.0, 1.0, st));
    POETX_TRY(bmm(dt, nb, b, b, b, q, true, n2, false, t3, 1.0, 0.0, st));
    POETX_TRY(bmm(dt, nb, b, b, b, q2, true, n2, false, t4, 1.0, 0.0, st));
    POETX_TRY(bmm(dt, nb, b, b, b, dg, false, q2, true, t5, 1.0, 0.0, st));
    POETX_TRY(bmm(dt, nb, b, b, b, n2, false, q2, true, t6, 1.0, 0.0, st));
    cnp_combine_bwd_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, dg, n2, t3, t4, t5, t6,
                                                                     dq);
    POETX_LAUNCHED("cnp_combine_bwd");
  } else {
    // generic adjoint (cnp.py:146-158): G = A S, A = I + Q, S = I + sum Q^i
    std::vector<T*> pw(k + 1, nullptr);  // pw[j] = Q^j, pw[0] unused (identity)
    for (int j = 1; j <= k; ++j) {
      pw[j] = ws.take<T>(n);
      POETX_REQUIRE(pw[j], POETX_ESHAPE, "cnp_backward: workspace too small");
    }
    T* series = ws.take<T>(n);
    T* ipq = ws.take<T>(n);
    T* ds = ws.take<T>(n);
    T* tmp = ws.take<T>(n);
    T* eye = ws.take<T>(n);
    POETX_REQUIRE(series && ipq && ds && tmp && eye, POETX_ESHAPE, "cnp_backward: workspace too small");
    cudaMemcpyAsync(pw[1], q, n * sizeof(T), cudaMemcpyDeviceToDevice, st);
    for (int j = 2; j <= k; ++j)
      POETX_TRY(bmm(dt, nb, b, b, b, pw[j - 1], false, q, false, pw[j], 1.0, 0.0, st));
    add_identity_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, b, nullptr, eye);
    POETX_LAUNCHED("add_identity");
    add_identity_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, b, q, ipq);
    POETX_LAUNCHED("add_identity");
    cudaMemcpyAsync(series, eye, n * sizeof(T), cudaMemcpyDeviceToDevice, st);
    for (int j = 1; j <= k; ++j) {
      accumulate_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(total, pw[j], series);
      POETX_LAUNCHED("accumulate");
    }
    POETX_TRY(bmm(dt, nb, b, b, b, dg, false, series, true, dq, 1.0, 0.0, st));  // dG S^T
    POETX_TRY(bmm(dt, nb, b, b, b, ipq, true, dg, false, ds, 1.0, 0.0, st));     // A^T dG
    for (int i = 1; i <= k; ++i) {
      for (int j = 0; j < i; ++j) {
        // dq += (Q^j)^T ds (Q^(i-1-j))^T
        const T* left = j == 0 ? eye : pw[j];
        const T* right = (i - 1 - j) == 0 ? eye : pw[i - 1 - j];
        POETX_TRY(bmm(dt, nb, b, b, b, left, true, ds, false, tmp, 1.0, 0.0, st));
        POETX_TRY(bmm(dt, nb, b, b, b, tmp, false, right, true, dq, 1.0, 1.0, st));
      }
    }
  }
  if (dpacked) POETX_TRY(pack_grad<T>(nb, b, dq, dpacked, accumulate, st));
  return POETX_OK;
}

// ----------------------------------------------------------- reductions ----
// deterministic two-stage sum of squares in double
template <typename T>
__global__ void sqdev_partial_kernel(int64_t total, int64_t b, const T* __restrict__ x,
                                     int subtract_identity, double* __restrict__ partial,
                                     int* __restrict__ nonfinite) {
  __shared__ double sh[256];
  double acc = 0.0;
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = static_cast<double>(Conv<T>::to_f(x[e]));
    if (subtract_identity) {
      int64_t r = e % (b * b);
      if (r / b == r % b) v -= 1.0;
    }
    if (!isfinite(v)) bad = 1;
    acc += v * v;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
  if (bad && nonfinite) *nonfinite = 1;
}

__global__ void sum_partials_kernel(int n, const double* __restrict__ partial, double* out,
                                    int do_sqrt, int accumulate) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double v = sh[0];
    if (accumulate) v += *out;
    *out = do_sqrt ? sqrt(v) : v;
  }
}

constexpr int kPartials = 512;

template <typename T>
static int sqdev(int64_t total, int64_t b, const void* x, int sub_eye, double* partial,
                 int* nonfinite, cudaStream_t st) {
  int grid = static_cast<int>(grid_for(total, 256, kPartials));
  sqdev_partial_kernel<T><<<grid, 256, 0, st>>>(total, b, static_cast<const T*>(x), sub_eye,
                                                partial, nonfinite);
  POETX_LAUNCHED("sqdev_partial");
  return grid;
}

// --------------------------------------------------------- permutations ----
template <typename T>
__global__ void permute_cols_kernel(int64_t rows, int64_t cols, const int32_t* __restrict__ idx,
                                    const T* __restrict__ x, T* __restrict__ y) {
  // one CTA per row (grid-stride over rows), threads over columns: coalesced
  // writes; reads gather within one row, which sits in L1/L2
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const T* xr = x + r * cols;
    T* yr = y + r * cols;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) yr[j] = xr[idx[j]];
  }
}

// BF16 feature permutation at HBM speed: each CTA stages whole rows in
// shared memory with 16-byte coalesced loads, then writes the permuted row
// with 16-byte coalesced stores, gathering 8 elements per store from smem
// (the index vector stays L1-resident across rows).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Feature-major tile gather: a tile of 8 token rows is staged TRANSPOSED in
// shared memory (one 16-byte slot per feature holding its 8 token values;
// slots XOR-swizzled within groups of 8 so the transposing stores are
// conflict-free), so gathering feature idx[j] for all 8 tokens is ONE
// 16-byte LDS instead of eight conflicted 2-byte LDS: the random accesses
// that bound the row-major kernel drop ~3x in smem wavefronts.  8x8 bf16
// transposes are 32 PRMTs in registers on the way in and out.

__global__ void __launch_bounds__(256) permute_cols_t8_kernel(int64_t rows, int cols,
                                                             const int32_t* __restrict__ idx,
                                                             const __nv_bfloat16* __restrict__ x,
                                                             __nv_bfloat16* __restrict__ y) {
  extern __shared__ __align__(16) uint4 slots[];  // [cols] x 16 B
  const int nv = cols / 8;
  const int64_t tiles = (rows + 7) / 8;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * 8;
    const int nr = static_cast<int>(rows - r0 < 8 ? rows - r0 : 8);
    for (int c = threadIdx.x; c < nv; c += blockDim.x) {
      uint4 rr[8], cc[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        rr[r] = r < nr ? __ldcs(reinterpret_cast<const uint4*>(x + (r0 + r) * cols) + c) : make_uint4(0, 0, 0, 0);
      tr8x8(rr, cc);
#pragma unroll
      for (int k = 0; k < 8; ++k) slots[fslot(8 * c + k)] = cc[k];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nv; c += blockDim.x) {
      const int4 i0 = __ldg(reinterpret_cast<const int4*>(idx) + 2 * c);
      const int4 i1 = __ldg(reinterpret_cast<const int4*>(idx) + 2 * c + 1);
      const int id[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
      uint4 g[8], o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) g[q] = slots[fslot(id[q])];
      tr8x8(g, o);  // g[q] = 8 tokens of feature id[q] -> o[r] = token r's 8 outputs
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < nr) __stcs(reinterpret_cast<uint4*>(y + (r0 + r) * cols) + c, o[r]);
    }
    __syncthreads();
  }
}

// rows are processed in chunks of R rows; chunk i+1 streams into the other
// smem buffer (cp.async) while chunk i is gathered and written
__global__ void __launch_bounds__(256) permute_cols_bf16_kernel(int64_t rows, int64_t cols, int R,
                                                              const int32_t* __restrict__ idx,
                                                              const __nv_bfloat16* __restrict__ x,
                                                              __nv_bfloat16* __restrict__ y) {
  extern __shared__ __align__(16) __nv_bfloat16 sbuf[];
  const int64_t nv = cols / 8;
  const int64_t chunk_elems = static_cast<int64_t>(R) * cols;
  const int64_t nchunks = (rows + R - 1) / R;
  auto issue = [&](int64_t c, int buf) {
    if (c < nchunks) {
      const int64_t r0 = c * R;
      const int64_t nr = rows - r0 < R ? rows - r0 : R;
      const uint4* src = reinterpret_cast<const uint4*>(x + r0 * cols);
      uint4* dst = reinterpret_cast<uint4*>(sbuf + buf * chunk_elems);
      for (int64_t i = threadIdx.x; i < nr * nv; i += blockDim.x) cp_async16(dst + i, src + i);
    }
    cp_async_commit();
  };
  int buf = 0;
  issue(blockIdx.x, 0);
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    issue(c + gridDim.x, buf ^ 1);
    cp_async_wait<1>();
    __syncthreads();
    const __nv_bfloat16* srow0 = sbuf + buf * chunk_elems;
    const int64_t r0 = c * R;
    const int64_t nr = rows - r0 < R ? rows - r0 : R;
    for (int64_t e = threadIdx.x; e < nr * nv; e += blockDim.x) {
      const int64_t rr = e / nv, i = e % nv;
      const __nv_bfloat16* srow = srow0 + rr * cols;
      const int4 ia = __ldg(reinterpret_cast<const int4*>(idx) + 2 * i);
      const int4 ib = __ldg(reinterpret_cast<const int4*>(idx) + 2 * i + 1);
      __nv_bfloat162 p0 = __halves2bfloat162(srow[ia.x], srow[ia.y]);
      __nv_bfloat162 p1 = __halves2bfloat162(srow[ia.z], srow[ia.w]);
      __nv_bfloat162 p2 = __halves2bfloat162(srow[ib.x], srow[ib.y]);
      __nv_bfloat162 p3 = __halves2bfloat162(srow[ib.z], srow[ib.w]);
      uint4 v;
      v.x = *reinterpret_cast<uint32_t*>(&p0);
      v.y = *reinterpret_cast<uint32_t*>(&p1);
      v.z = *reinterpret_cast<uint32_t*>(&p2);
      v.w = *reinterpret_cast<uint32_t*>(&p3);
      __stcs(reinterpret_cast<uint4*>(y + (r0 + rr) * cols) + i, v);
    }
    __syncthreads();
    buf ^= 1;
  }
  cp_async_wait<0>();
}

template <typename T>
__global__ void gather2d_kernel(int64_t rows, int64_t cols, const int32_t* __restrict__ ridx,
                                const int32_t* __restrict__ cidx, const T* __restrict__ x,
                                T* __restrict__ y) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const T* xr = x + static_cast<int64_t>(ridx ? ridx[r] : r) * cols;
    T* yr = y + r * cols;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) yr[j] = xr[cidx ? cidx[j] : j];
  }
}

template <typename T>
static int gather2d_t(int64_t rows, int64_t cols, const int32_t* ridx, const int32_t* cidx,
                      const void* x, void* y, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return POETX_OK;
  unsigned grid = static_cast<unsigned>(rows < 148 * 16 ? rows : 148 * 16);
  if constexpr (sizeof(T) == 2) {
    static const int t8 = [] {
      const char* e = getenv("POETX_PERMUTE_T8");
      return e && e[0] == '0' ? 0 : 1;
    }();
    const size_t tsm = static_cast<size_t>(cols) * 16;
    if (t8 && ridx == nullptr && cidx != nullptr && cols % 8 == 0 && tsm <= 200 * 1024 && cols < INT32_MAX &&
        ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
          reinterpret_cast<uintptr_t>(cidx)) & 15) == 0) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(permute_cols_t8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
      }
      const int64_t tiles = (rows + 7) / 8;
      int per_sm = static_cast<int>((228 * 1024) / (tsm + 1024));
      if (per_sm > 8) per_sm = 8;
      if (per_sm < 1) per_sm = 1;
      const int64_t cap = 148LL * per_sm;
      permute_cols_t8_kernel<<<static_cast<unsigned>(tiles < cap ? tiles : cap), 256, tsm, st>>>(
          rows, static_cast<int>(cols), cidx, reinterpret_cast<const __nv_bfloat16*>(x),
          reinterpret_cast<__nv_bfloat16*>(y));
      POETX_LAUNCHED("permute_cols_t8");
      return POETX_OK;
    }
    // chunk of R rows ~ 12 KB, two buffers per CTA
    int R = static_cast<int>((12 * 1024) / (cols * 2));
    if (R < 1) R = 1;
    const size_t smem = 2 * static_cast<size_t>(R) * cols * 2;
    if (ridx == nullptr && cidx != nullptr && cols % 8 == 0 && smem <= 100 * 1024 &&
        ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
          reinterpret_cast<uintptr_t>(cidx)) & 15) == 0) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(permute_cols_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             100 * 1024);
        attr = true;
      }
      int64_t chunks = (rows + R - 1) / R;
      unsigned g = static_cast<unsigned>(chunks < 148 * 6 ? chunks : 148 * 6);
      permute_cols_bf16_kernel<<<g, 256, smem, st>>>(rows, cols, R, cidx,
                                                      reinterpret_cast<const __nv_bfloat16*>(x),
                                                      reinterpret_cast<__nv_bfloat16*>(y));
      POETX_LAUNCHED("permute_cols_bf16");
      return POETX_OK;
    }
  }
  if (ridx == nullptr && cidx != nullptr) {
    permute_cols_kernel<T><<<grid, 256, 0, st>>>(rows, cols, cidx, static_cast<const T*>(x),
                                                  static_cast<T*>(y));
    POETX_LAUNCHED("permute_cols");
  } else {
    gather2d_kernel<T><<<grid, 256, 0, st>>>(rows, cols, ridx, cidx, static_cast<const T*>(x),
                                              static_cast<T*>(y));
    POETX_LAUNCHED("gather2d");
  }
  return POETX_OK;
}

int gather2d(int dt, int64_t rows, int64_t cols, const int32_t* ridx, const int32_t* cidx,
             const void* x, void* y, cudaStream_t st) {
  switch (dt) {
    case POETX_F32: return gather2d_t<float>(rows, cols, ridx, cidx, x, y, st);
    case POETX_F64: return gather2d_t<double>(rows, cols, ridx, cidx, x, y, st);
    case POETX_BF16: return gather2d_t<__nv_bfloat16>(rows, cols, ridx, cidx, x, y, st);
  }
  set_error("gather2d: bad dtype %d", dt);
  return POETX_ESHAPE;
}

// ------------------------------------------------------- block-diagonal ----
int apply_features(int dt, int64_t T, int64_t nb, int64_t b, const void* g, int transpose,
                   const void* x, void* y, cudaStream_t st) {
  const int64_t dim = nb * b;
  if (T <= 0 || nb <= 0) return POETX_OK;
  GemmDesc d{};
  d.M = T; d.N = b; d.K = b; d.batch = nb;
  d.A = x; d.sAb = b; d.sAm = dim; d.sAk = 1;
  d.B = g; d.sBb = b * b; d.sBk = transpose ? 1 : b; d.sBn = transpose ? b : 1;
  d.C = y; d.sCb = b; d.sCm = dim; d.sCn = 1;
  d.alpha = 1.0; d.beta = 0.0;
  if (dt == POETX_BF16 && tc_enabled()) {
    int rc = tc_blockdiag(d, st);
    if (rc != POETX_ENOTSUPPORTED) return rc;
  }
  return gemm(dt, dt, d, st);
}

// POET-XQ: y[s-rows, :] = g[s] (codes[s-rows, :] * scales[s-rows]) with the
// int8 codes dequantized inside the pair GEMM's producer (bf16 g, bf16 y)
int apply_weight_rows_q8(int64_t nb, int64_t b, int64_t cols, const void* g, const int8_t* codes,
                         const float* scales, void* y, cudaStream_t st) {
  if (nb <= 0 || cols <= 0) return POETX_OK;
  if (!tc_enabled() || b != 256 || cols % 256) return POETX_ENOTSUPPORTED;
  TcOperand A{g, nb * b, b, b, false};
  TcOperand B{codes, nb * b, cols, cols, true, scales};
  TcProblem p{};
  p.M = b; p.N = cols; p.K = b; p.groups = static_cast<int>(nb); p.splits = 1;
  p.bn = 256;
  p.a_g1 = static_cast<int>(b);
  p.b_g1 = static_cast<int>(b);
  p.C = y; p.ldc = cols; p.c_goff = b * cols;
  p.alpha = 1.0f; p.name = "tc_wfold_q8"; p.tma_epi = 1;
  return tc_grouped(A, B, p, st);
}

// POET-XQ: y = W1^T [n, m] for W1 = PM bd(G_P), with the codes dequantized in
// the pair GEMM's producer: y[t*b + i, j] = sum_k G_P[t][k, i] PM[j, t*b + k]
// (A = G_P[t] read MN-major, B = the b code columns of block t, K-major, one
// scale per PM row j).  The adjoint then reads y as its K x N operand.
int apply_weight_cols_t_q8(int64_t m, int64_t nb, int64_t b, const void* g_p, const int8_t* codes,
                           const float* scales, void* y, cudaStream_t st) {
  if (nb <= 0 || m <= 0) return POETX_OK;
  if (!tc_enabled() || b != 256 || m % 256) return POETX_ENOTSUPPORTED;
  TcOperand A{g_p, nb * b, b, b, true};
  TcOperand B{codes, m, nb * b, nb * b, false, scales};
  TcProblem p{};
  p.M = b; p.N = m; p.K = b; p.groups = static_cast<int>(nb); p.splits = 1;
  p.bn = 256;
  p.a_g1 = static_cast<int>(b);
  p.b_g0 = static_cast<int>(b);
  p.C = y; p.ldc = m; p.c_goff = b * m;
  p.alpha = 1.0f; p.name = "tc_wfold_t_q8"; p.tma_epi = 1;
  return tc_grouped(A, B, p, st);
}

int apply_weight_rows(int dt, int64_t nb, int64_t b, int64_t cols, const void* g, int transpose,
                      const void* w, void* y, cudaStream_t st) {
  if (nb <= 0 || cols <= 0) return POETX_OK;
  if (dt == POETX_BF16 && tc_enabled() && !transpose && b % 64 == 0 && b <= 256 && cols % 256 == 0) {
    // y[s-rows, :] = g[s] w[s-rows, :] as a grouped tcgen05 product:
    // A = g[s] (K-major), B = the b rows of w (MN-major), one group per block
    TcOperand A{g, nb * b, b, b, false};
    TcOperand B{w, nb * b, cols, cols, true};
    TcProblem p{};
    p.M = b; p.N = cols; p.K = b; p.groups = static_cast<int>(nb); p.splits = 1;
    p.bn = static_cast<int>(b < 256 ? b : 256);
    p.a_g1 = static_cast<int>(b);
    p.b_g1 = static_cast<int>(b);
    p.C = y; p.ldc = cols; p.c_goff = b * cols;
    p.alpha = 1.0f; p.name = "tc_wfold"; p.tma_epi = 1;
    int rc = tc_grouped(A, B, p, st);
    if (rc != POETX_ENOTSUPPORTED) return rc;
  }
  GemmDesc d{};
  d.M = b; d.N = cols; d.K = b; d.batch = nb;
  d.A = g; d.sAb = b * b; d.sAm = transpose ? 1 : b; d.sAk = transpose ? b : 1;
  d.B = w; d.sBb = b * cols; d.sBk = cols; d.sBn = 1;
  d.C = y; d.sCb = b * cols; d.sCm = cols; d.sCn = 1;
  d.alpha = 1.0; d.beta = 0.0;
  return gemm(dt, dt, d, st);
}

template <typename T>
__global__ void reduce_splits_kernel(int64_t total, int splits, const T* __restrict__ part,
                                     T* __restrict__ out, int accumulate) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    T acc = part[e];
    for (int s = 1; s < splits; ++s) acc = acc + part[s * total + e];  // fixed order
    out[e] = accumulate ? out[e] + acc : acc;
  }
}

// fp32, 4 elements per thread, partials read with streaming loads (same fixed order)
__global__ void reduce_splits_f4_kernel(int64_t total4, int splits, const float4* __restrict__ part,
                                        float4* __restrict__ out, int accumulate) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total4;
       e += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = __ldcs(part + e);
    for (int s = 1; s < splits; ++s) {
      const float4 v = __ldcs(part + s * total4 + e);
      acc.x = acc.x + v.x; acc.y = acc.y + v.y; acc.z = acc.z + v.z; acc.w = acc.w + v.w;
    }
    if (accumulate) {
      const float4 o = out[e];
      acc.x = o.x + acc.x; acc.y = o.y + acc.y; acc.z = o.z + acc.z; acc.w = o.w + acc.w;
    }
    out[e] = acc;
  }
}

static int outer_splits(int64_t T, int64_t nb, int64_t b) {
  int64_t tiles = nb * ((b + 63) / 64) * ((b + 63) / 64);
  int64_t want = (2 * 148 + tiles - 1) / tiles;
  int64_t maxs = T / 256;
  if (want > maxs) want = maxs;
  if (want < 1) want = 1;
  if (want > 64) want = 64;
  return static_cast<int>(want);
}

size_t outer_ws_bytes(int dt, int64_t T, int64_t nb, int64_t b) {
  int s = outer_splits(T, nb, b);
  size_t acc = dt == POETX_F64 ? 8 : 4;
  return s > 1 ? align_up(static_cast<size_t>(s) * nb * b * b * acc) : 0;
}

int segmented_outer(int dt, int64_t T, int64_t nb, int64_t b, const void* x, const void* y,
                    void* out, int accumulate, Workspace& ws, cudaStream_t st) {
  const int64_t dim = nb * b, total = nb * b * b;
  const int out_dt = dt == POETX_F64 ? POETX_F64 : POETX_F32;
  const size_t acc_sz = out_dt == POETX_F64 ? 8 : 4;
  if (nb <= 0 || b <= 0) return POETX_OK;
  if (dt == POETX_BF16 && tc_enabled() && b % 64 == 0 && dim % 8 == 0 && T > 0) {
    // tcgen05: both operands MN-major (tokens are the contraction index),
    // deterministic split-T partials reduced in fixed order
    const int s = tc_outer_splits(T, nb, b);
    float* tgt = static_cast<float*>(out);
    if (s > 1 || accumulate) {
      tgt = static_cast<float*>(ws.take_bytes(static_cast<size_t>(s) * total * 4));
      POETX_REQUIRE(tgt, POETX_ESHAPE, "segmented_outer: workspace too small");
    }
    TcOperand xa{x, T, dim, dim, true};
    TcOperand yb{y, T, dim, dim, true};
    TcProblem p{};
    p.M = b; p.N = b; p.K = T; p.groups = static_cast<int>(nb); p.splits = s;
    p.bn = static_cast<int>(b < 256 ? b : 256);
    p.a_g0 = static_cast<int>(b); p.b_g0 = static_cast<int>(b);
    p.C = tgt; p.ldc = b; p.c_goff = b * b; p.c_soff = total; p.out_f32 = 1; p.alpha = 1.0f;
    p.name = "tc_outer";
    p.ms = 1;  // (ms = 2 halves B traffic but doubles split-K partials: measured slower)
    p.tma_epi = 1;
    int rc = tc_grouped(xa, yb, p, st);
    if (rc != POETX_ENOTSUPPORTED) {
      POETX_TRY(rc);
      if (tgt != out) {
        if (total % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
          reduce_splits_f4_kernel<<<grid_for(total / 4, 256), 256, 0, st>>>(
              total / 4, s, reinterpret_cast<const float4*>(tgt), static_cast<float4*>(out), accumulate);
        } else {
          reduce_splits_kernel<float><<<grid_for(total, 256), 256, 0, st>>>(
              total, s, tgt, static_cast<float*>(out), accumulate);
        }
        POETX_LAUNCHED("reduce_splits");
      }
      return POETX_OK;
    }
  }
  int splits = outer_splits(T, nb, b);
  int64_t chunk = (T + splits - 1) / splits;
  void* part = out;
  if (splits > 1 || accumulate) {
    part = ws.take_bytes(static_cast<size_t>(splits) * total * acc_sz);
    POETX_REQUIRE(part, POETX_ESHAPE, "segmented_outer: workspace too small");
  }
  const size_t xe = elt_size(dt);
  for (int s = 0; s < splits; ++s) {
    int64_t t0 = s * chunk, t1 = t0 + chunk < T ? t0 + chunk : T;
    GemmDesc d{};
    d.M = b; d.N = b; d.K = t1 > t0 ? t1 - t0 : 0; d.batch = nb;
    d.A = static_cast<const char*>(x) + t0 * dim * xe; d.sAb = b; d.sAm = 1; d.sAk = dim;
    d.B = static_cast<const char*>(y) + t0 * dim * xe; d.sBb = b; d.sBk = dim; d.sBn = 1;
    d.C = static_cast<char*>(part) + s * total * acc_sz; d.sCb = b * b; d.sCm = b; d.sCn = 1;
    d.alpha = 1.0; d.beta = 0.0;
    POETX_TRY(gemm(dt, out_dt, d, st));
  }
  if (part != out) {
    if (out_dt == POETX_F64)
      reduce_splits_kernel<double><<<grid_for(total, 256), 256, 0, st>>>(
          total, splits, static_cast<const double*>(part), static_cast<double*>(out), accumulate);
    else
      reduce_splits_kernel<float><<<grid_for(total, 256), 256, 0, st>>>(
          total, splits, static_cast<const float*>(part), static_cast<float*>(out), accumulate);
    POETX_LAUNCHED("reduce_splits");
  }
  return POETX_OK;
}

// ----------------------------------------------------------------- AdamW ----
// Reference operation order (optim.py:139-148), no FMA contraction:
//   m = m*b1 + (1-b1)*g ; v = v*b2 + ((1-b2)*g)*g ;
//   mhat = m/bc1 ; vhat = v/bc2 ; p = p*(1-lr*wd) ; p = p - (lr*mhat)/(sqrt(vhat)+eps)
struct AdamScalars {
  double lr, b1, b2, eps, lrwd, bc1, bc2, thr;
};

__device__ __forceinline__ float op_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float op_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float op_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float op_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float op_sqrt(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double op_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double op_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double op_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double op_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double op_sqrt(double a) { return __dsqrt_rn(a); }

template <typename T>
__global__ void adamw_kernel(int64_t n, T* __restrict__ p, T* __restrict__ g, T* __restrict__ m,
                             T* __restrict__ v, AdamScalars s, const double* __restrict__ sqnorm,
                             int write_back, const double* __restrict__ dyn) {
  if (dyn) {  // step-dependent scalars from device memory (CUDA-graph replays)
    s.lr = dyn[0];
    s.lrwd = dyn[1];
    s.bc1 = dyn[2];
    s.bc2 = dyn[3];
    s.thr = dyn[4];
  }
  const T b1 = static_cast<T>(s.b1), b2 = static_cast<T>(s.b2), one = T(1);
  const T omb1 = op_sub(one, b1), omb2 = op_sub(one, b2);
  const T bc1 = static_cast<T>(s.bc1), bc2 = static_cast<T>(s.bc2);
  const T decay = op_sub(one, static_cast<T>(s.lrwd)), lr = static_cast<T>(s.lr);
  const T eps = static_cast<T>(s.eps);
  bool clip = false;
  T factor = one;
  if (sqnorm) {
    double norm = sqrt(*sqnorm);
    // a non-finite gradient norm aborts the step in the reference
    // (optim.py:87-89); on the device (no host sync, CUDA-graph replays) the
    // update is skipped so parameters and moments stay intact, and the
    // caller raises NumericsError from the norm kernel's flag
    if (!isfinite(norm)) return;
    if (norm > s.thr && norm > 0.0) {  // optim.py:90-93
      clip = true;
      factor = static_cast<T>(s.thr / norm);
    }
  }
  auto update = [&](T& pi_, T& gi_, T& mi_, T& vi_) {
    T gi = gi_;
    if (clip) gi = op_mul(gi, factor);
    const T mi = op_add(op_mul(mi_, b1), op_mul(omb1, gi));
    const T vi = op_add(op_mul(vi_, b2), op_mul(op_mul(omb2, gi), gi));
    const T mhat = op_div(mi, bc1), vhat = op_div(vi, bc2);
    T pi = op_mul(pi_, decay);
    pi_ = op_sub(pi, op_div(op_mul(lr, mhat), op_add(op_sqrt(vhat), eps)));
    gi_ = gi;
    mi_ = mi;
    vi_ = vi;
  };
  // 16-byte vectors (same per-element operation order, so bitwise identical)
  constexpr int V = 16 / sizeof(T);
  using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                        reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  int64_t done = 0;
  if (vec_ok) {
    const int64_t nv = n / V;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
      Vec pv = reinterpret_cast<Vec*>(p)[i], gv = reinterpret_cast<Vec*>(g)[i];
      Vec mv = reinterpret_cast<Vec*>(m)[i], vv = reinterpret_cast<Vec*>(v)[i];
      T* pp = reinterpret_cast<T*>(&pv);
      T* gg = reinterpret_cast<T*>(&gv);
      T* mm = reinterpret_cast<T*>(&mv);
      T* ww = reinterpret_cast<T*>(&vv);
#pragma unroll
      for (int q = 0; q < V; ++q) update(pp[q], gg[q], mm[q], ww[q]);
      reinterpret_cast<Vec*>(p)[i] = pv;
      reinterpret_cast<Vec*>(m)[i] = mv;
      reinterpret_cast<Vec*>(v)[i] = vv;
      if (clip && write_back) reinterpret_cast<Vec*>(g)[i] = gv;
    }
    done = nv * V;
  }
  for (int64_t i = done + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    T pi = p[i], gi = g[i], mi = m[i], vi = v[i];
    update(pi, gi, mi, vi);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (clip && write_back) g[i] = gi;
  }
}

}  // namespace poetx

using namespace poetx;

// ================================================================ C ABI =====
extern "C" {

const char* poetx_last_error(void) { return g_last_error.c_str(); }
int poetx_abi_version(void) { return POETX_ABI_VERSION; }
uint64_t poetx_launch_count(void) { return launch_counter().load(); }

int poetx_skew_from_packed(int dtype, int64_t nb, int64_t b, const void* packed, void* q,
                           void* stream) {
  POETX_REQUIRE(nb >= 0 && b >= 1, POETX_ESHAPE, "bad block layout (%lld, %lld)", (long long)nb,
                (long long)b);
  if (dtype == POETX_F32) return skew_unpack<float>(nb, b, packed, q, as_stream(stream));
  if (dtype == POETX_F64) return skew_unpack<double>(nb, b, packed, q, as_stream(stream));
  set_error("skew_from_packed: dtype must be F32 or F64");
  return POETX_ESHAPE;
}

int poetx_packed_grad_from_skew_grad(int dtype, int64_t nb, int64_t b, const void* dq, void* g,
                                     int accumulate, void* stream) {
  POETX_REQUIRE(nb >= 0 && b >= 1, POETX_ESHAPE, "bad block layout");
  if (dtype == POETX_F32) return pack_grad<float>(nb, b, dq, g, accumulate, as_stream(stream));
  if (dtype == POETX_F64) return pack_grad<double>(nb, b, dq, g, accumulate, as_stream(stream));
  set_error("packed_grad_from_skew_grad: dtype must be F32 or F64");
  return POETX_ESHAPE;
}

size_t poetx_cnp_workspace_bytes(int dtype, int64_t nb, int64_t b, int k) {
  return cnp_ws_bytes(dtype, nb, b, k);
}

int poetx_cnp_forward(int dtype, int64_t nb, int64_t b, int k, const void* q, const void* packed,
                      void* g, void* g_bf16, void* q2, void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(k >= 1, POETX_ECONFIG, "neumann_k must be >= 1, got %d", k);
  POETX_REQUIRE(nb >= 1 && b >= 1, POETX_ESHAPE, "bad block layout (%lld, %lld)", (long long)nb,
                (long long)b);
  POETX_REQUIRE(g != nullptr && (q != nullptr || packed != nullptr), POETX_ESHAPE,
                "cnp_forward: null operand");
  Workspace w(ws, ws_bytes);
  if (dtype == POETX_F32)
    return cnp_forward_t<float>(dtype, nb, b, k, q, packed, g, g_bf16, q2, w, as_stream(stream));
  if (dtype == POETX_F64)
    return cnp_forward_t<double>(dtype, nb, b, k, q, packed, g, g_bf16, q2, w, as_stream(stream));
  set_error("cnp_forward: dtype must be F32 or F64");
  return POETX_ESHAPE;
}

int poetx_cnp_backward(int dtype, int64_t nb, int64_t b, int k, const void* q, const void* packed,
                       const void* q2, const void* dg, void* dq, void* dpacked, int accumulate,
                       void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(k >= 1, POETX_ECONFIG, "neumann_k must be >= 1, got %d", k);
  POETX_REQUIRE(nb >= 1 && b >= 1, POETX_ESHAPE, "bad block layout");
  POETX_REQUIRE(dg != nullptr && (q != nullptr || packed != nullptr), POETX_ESHAPE,
                "cnp_backward: null operand");
  Workspace w(ws, ws_bytes);
  if (dtype == POETX_F32)
    return cnp_backward_t<float>(dtype, nb, b, k, q, packed, q2, dg, dq, dpacked, accumulate, w,
                                 as_stream(stream));
  if (dtype == POETX_F64)
    return cnp_backward_t<double>(dtype, nb, b, k, q, packed, q2, dg, dq, dpacked, accumulate, w,
                                  as_stream(stream));
  set_error("cnp_backward: dtype must be F32 or F64");
  return POETX_ESHAPE;
}

int poetx_orthogonality_error(int dtype, int64_t nb, int64_t b, const void* g, double* out,
                              void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(dtype == POETX_F32 || dtype == POETX_F64, POETX_ESHAPE,
                "orthogonality_error: dtype must be F32 or F64");
  cudaStream_t st = as_stream(stream);
  Workspace w(ws, ws_bytes);
  const int64_t total = nb * b * b;
  void* gtg = w.take_bytes(static_cast<size_t>(total) * elt_size(dtype));
  double* part = w.take<double>(kPartials);
  POETX_REQUIRE(gtg && part, POETX_ESHAPE, "orthogonality_error: workspace too small");
  POETX_TRY(bmm(dtype, nb, b, b, b, g, true, g, false, gtg, 1.0, 0.0, st));
  int parts = dtype == POETX_F32 ? sqdev<float>(total, b, gtg, 1, part, nullptr, st)
                                 : sqdev<double>(total, b, gtg, 1, part, nullptr, st);
  if (parts < 0) return parts;
  sum_partials_kernel<<<1, 256, 0, st>>>(parts, part, out, 1, 0);
  POETX_LAUNCHED("sum_partials");
  return POETX_OK;
}

int poetx_permute_cols(int dtype, int64_t rows, int64_t cols, const int32_t* idx, const void* x,
                       void* y, void* stream) {
  POETX_REQUIRE(rows >= 0 && cols >= 0 && idx, POETX_ESHAPE, "permute_cols: bad arguments");
  return gather2d(dtype, rows, cols, nullptr, idx, x, y, as_stream(stream));
}
int poetx_permute_rows(int dtype, int64_t rows, int64_t cols, const int32_t* idx, const void* x,
                       void* y, void* stream) {
  POETX_REQUIRE(rows >= 0 && cols >= 0 && idx, POETX_ESHAPE, "permute_rows: bad arguments");
  return gather2d(dtype, rows, cols, idx, nullptr, x, y, as_stream(stream));
}
int poetx_gather2d(int dtype, int64_t rows, int64_t cols, const int32_t* ridx, const int32_t* cidx,
                   const void* x, void* y, void* stream) {
  POETX_REQUIRE(rows >= 0 && cols >= 0, POETX_ESHAPE, "gather2d: bad arguments");
  return gather2d(dtype, rows, cols, ridx, cidx, x, y, as_stream(stream));
}

int poetx_apply_to_features(int dtype, int64_t T, int64_t nb, int64_t b, const void* g,
                            int transpose, const void* x, void* y, void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "apply_to_features: bad dtype");
  POETX_REQUIRE(T >= 0 && nb >= 1 && b >= 1, POETX_ESHAPE, "apply_to_features: bad shape");
  return apply_features(dtype, T, nb, b, g, transpose, x, y, as_stream(stream));
}
int poetx_apply_to_weight_rows(int dtype, int64_t nb, int64_t b, int64_t cols, const void* g,
                               int transpose, const void* w, void* y, void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "apply_to_weight_rows: bad dtype");
  return apply_weight_rows(dtype, nb, b, cols, g, transpose, w, y, as_stream(stream));
}
size_t poetx_segmented_outer_workspace_bytes(int dtype, int64_t T, int64_t nb, int64_t b) {
  size_t acc = dtype == POETX_F64 ? 8 : 4;
  return outer_ws_bytes(dtype, T, nb, b) + align_up(static_cast<size_t>(nb * b * b) * acc) +
         tc_outer_ws_bytes(T, nb, b) + 4096;
}
int poetx_segmented_outer(int dtype, int64_t T, int64_t nb, int64_t b, const void* x,
                          const void* y, void* out, int accumulate, void* ws, size_t ws_bytes,
                          void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "segmented_outer: bad dtype");
  POETX_REQUIRE(T >= 0 && nb >= 1 && b >= 1, POETX_ESHAPE, "segmented_outer: bad shape");
  Workspace w(ws, ws_bytes);
  return segmented_outer(dtype, T, nb, b, x, y, out, accumulate, w, as_stream(stream));
}

int poetx_matmul(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                 int transA, const void* B, int64_t ldb, int transB, void* C, int64_t ldc,
                 int accumulate, void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "matmul: bad dtype");
  POETX_REQUIRE(M >= 0 && N >= 0 && K >= 0, POETX_ESHAPE, "matmul: negative shape");
  cudaStream_t st = as_stream(stream);
  if (dtype == POETX_BF16 && tc_enabled() && !accumulate) {
    int rc = tc_matmul(M, N, K, A, lda, transA, B, ldb, transB, C, ldc, st);
    if (rc != POETX_ENOTSUPPORTED) return rc;
  }
  GemmDesc d{};
  d.M = M; d.N = N; d.K = K; d.batch = 1;
  d.A = A; d.sAb = 0; d.sAm = transA ? 1 : lda; d.sAk = transA ? lda : 1;
  d.B = B; d.sBb = 0; d.sBk = transB ? 1 : ldb; d.sBn = transB ? ldb : 1;
  d.C = C; d.sCb = 0; d.sCm = ldc; d.sCn = 1;
  d.alpha = 1.0; d.beta = accumulate ? 1.0 : 0.0;
  return gemm(dtype, dtype, d, st);
}

int poetx_matmul_q8(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const int8_t* codes, int64_t ldb,
                    int transB, const float* scales, void* C, int64_t ldc, void* stream) {
  POETX_REQUIRE(M >= 0 && N >= 0 && K >= 0 && A && codes && scales && C, POETX_ESHAPE, "matmul_q8: bad arguments");
  const int rc = tc_enabled() ? tc_matmul_q8(M, N, K, A, lda, 0, codes, ldb, transB, scales, C, ldc, as_stream(stream))
                              : POETX_ENOTSUPPORTED;
  POETX_REQUIRE(rc != POETX_ENOTSUPPORTED, POETX_ESHAPE,
                "matmul_q8: shape not handled by the fused int8 pair GEMM (N %% 256, 16-byte pitches)");
  return rc;
}

size_t poetx_sqnorm_workspace_bytes(int ntensors, const int64_t* numel) {
  (void)numel;
  return align_up(static_cast<size_t>(ntensors + 1) * kPartials * sizeof(double)) + 4096;
}

int poetx_sqnorm(int dtype, int ntensors, const void* const* g, const int64_t* numel, double* out,
                 int* nonfinite, void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(dtype == POETX_F32 || dtype == POETX_F64, POETX_ESHAPE, "sqnorm: bad dtype");
  cudaStream_t st = as_stream(stream);
  Workspace w(ws, ws_bytes);
  double* part = w.take<double>(static_cast<size_t>(ntensors + 1) * kPartials);
  POETX_REQUIRE(part, POETX_ESHAPE, "sqnorm: workspace too small");
  if (nonfinite) cudaMemsetAsync(nonfinite, 0, sizeof(int), st);
  cudaMemsetAsync(out, 0, sizeof(double), st);
  for (int i = 0; i < ntensors; ++i) {
    if (numel[i] <= 0) continue;
    int parts = dtype == POETX_F32 ? sqdev<float>(numel[i], 1, g[i], 0, part, nonfinite, st)
                                   : sqdev<double>(numel[i], 1, g[i], 0, part, nonfinite, st);
    sum_partials_kernel<<<1, 256, 0, st>>>(parts, part, out, 0, 1);
    POETX_LAUNCHED("sum_partials");
  }
  return POETX_OK;
}

static int adamw_launch(int dtype, int ntensors, void* const* p, void* const* g, void* const* m,
                        void* const* v, const int64_t* numel, const AdamScalars& s,
                        const double* sqnorm, int write_back_grads, const double* dyn,
                        cudaStream_t st);

int poetx_adamw_dyn(int dtype, int ntensors, void* const* p, void* const* g, void* const* m,
                    void* const* v, const int64_t* numel, double beta1, double beta2, double eps,
                    const double* dyn, const double* sqnorm, int write_back_grads, void* stream) {
  POETX_REQUIRE(dtype == POETX_F32 || dtype == POETX_F64, POETX_ESHAPE, "adamw: bad dtype");
  POETX_REQUIRE(dyn != nullptr, POETX_ESHAPE, "adamw_dyn: null scalars");
  AdamScalars s{0.0, beta1, beta2, eps, 0.0, 1.0, 1.0, 0.0};
  return adamw_launch(dtype, ntensors, p, g, m, v, numel, s, sqnorm, write_back_grads, dyn,
                      as_stream(stream));
}

int poetx_adamw(int dtype, int ntensors, void* const* p, void* const* g, void* const* m,
                void* const* v, const int64_t* numel, double lr, double beta1, double beta2,
                double eps, double weight_decay, double bc1, double bc2, const double* sqnorm,
                double clip_threshold, int write_back_grads, void* stream) {
  POETX_REQUIRE(dtype == POETX_F32 || dtype == POETX_F64, POETX_ESHAPE, "adamw: bad dtype");
  AdamScalars s{lr, beta1, beta2, eps, lr * weight_decay, bc1, bc2, clip_threshold};
  return adamw_launch(dtype, ntensors, p, g, m, v, numel, s, sqnorm, write_back_grads, nullptr,
                      as_stream(stream));
}

static int adamw_launch(int dtype, int ntensors, void* const* p, void* const* g, void* const* m,
                        void* const* v, const int64_t* numel, const AdamScalars& s,
                        const double* sqnorm, int write_back_grads, const double* dyn,
                        cudaStream_t st) {
  for (int i = 0; i < ntensors; ++i) {
    if (numel[i] <= 0) continue;
    unsigned grid = grid_for((numel[i] + 3) / 4, 256, 148 * 16);
    if (dtype == POETX_F32)
      adamw_kernel<float><<<grid, 256, 0, st>>>(numel[i], static_cast<float*>(p[i]),
                                                 static_cast<float*>(g[i]), static_cast<float*>(m[i]),
                                                 static_cast<float*>(v[i]), s, sqnorm,
                                                 write_back_grads, dyn);
    else
      adamw_kernel<double><<<grid, 256, 0, st>>>(numel[i], static_cast<double*>(p[i]),
                                                  static_cast<double*>(g[i]),
                                                  static_cast<double*>(m[i]),
                                                  static_cast<double*>(v[i]), s, sqnorm,
                                                  write_back_grads, dyn);
    POETX_LAUNCHED("adamw");
  }
  return POETX_OK;
}

}  // extern "C"
