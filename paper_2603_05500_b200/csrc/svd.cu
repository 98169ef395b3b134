// Singular values by one-sided Jacobi rotations on the device, float64 --
// the reference's svd_singular_values (linalg.py:166-218) that its spectrum
// audit (runner.py:452-529), spectral_norm (linalg.py:221-224) and the
// merge-time sv-drift (layer.py:296-299) are built on.
//
// Same rotation and stopping rule as the reference: for a column pair (p, q)
// with squared norms alpha, beta and correlation gamma, skip when
// |gamma| <= tol sqrt(alpha beta), else rotate by the classic Jacobi angle
// (zeta = (beta - alpha) / 2 gamma) and recompute both norms from the new
// columns; stop after the first sweep without a rotation, or report
// non-convergence with the worst relative off-diagonal of the last sweep.
// The pair ORDER differs: the reference sweeps (p, q) lexicographically, one
// pair at a time; here each sweep is n-1 rounds of the round-robin
// (circle-method) schedule, whose n/2 disjoint pairs per round run on the
// CTA's warps in parallel.  Converged singular values agree to the tolerance,
// not bit for bit.
//
// One CTA per matrix (batched: the audit's stack of b x b skew blocks runs in
// one launch); the tall working copy lives column-major in the workspace,
// the squared column norms in shared memory.
#include "common.cuh"

namespace poetx {
namespace {

constexpr int SV_THREADS = 256, SV_WARPS = SV_THREADS / 32;
constexpr int64_t SV_MAX_COLS = 4096;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// tall column-major working copy: W[c * m + r] of the [m x n] (m >= n) matrix
// a (rows >= cols) or a^T (rows < cols)
__global__ void sv_prep_kernel(int64_t batch, int64_t rows, int64_t cols, const double* __restrict__ a,
                               double* __restrict__ w) {
  const int64_t per = rows * cols, total = batch * per;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / per, e = i % per;
    if (rows >= cols) {  // i enumerates w: column c = e / rows, row r = e % rows of a
      const int64_t c = e / rows, r = e % rows;
      w[i] = a[b * per + r * cols + c];
    } else {  // columns of a^T are the rows of a: a straight copy
      w[i] = a[i];
    }
  }
}

__global__ void __launch_bounds__(SV_THREADS) jacobi_sv_kernel(int64_t m, int64_t n, double* __restrict__ W, double tol,
                                                               int max_sweeps, double* __restrict__ sv,
                                                               double* __restrict__ resid, int* __restrict__ sweeps) {
  extern __shared__ double norms[];  // [n]
  __shared__ int rotated;
  __shared__ double wmax[SV_WARPS];
  double* A = W + static_cast<int64_t>(blockIdx.x) * m * n;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n2 = static_cast<int>(n + (n & 1));  // even: one dummy column when n is odd

  for (int64_t c = warp; c < n; c += SV_WARPS) {
    const double* col = A + c * m;
    double s = 0.0;
    for (int64_t r = lane; r < m; r += 32) s += col[r] * col[r];
    s = warp_sum_d(s);
    if (lane == 0) norms[c] = s;
  }
  __syncthreads();

  int used = -1;
  double worst = 0.0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    double wl = 0.0;
    __syncthreads();
    for (int k = 0; k < n2 - 1; ++k) {
      for (int i = warp; i < n2 / 2; i += SV_WARPS) {
        // circle method: column n2-1 fixed, the others rotate by one per round
        int p, q;
        if (i == 0) {
          p = k;
          q = n2 - 1;
        } else {
          p = (k + i) % (n2 - 1);
          q = (k - i + (n2 - 1)) % (n2 - 1);
        }
        if (p > q) { const int t = p; p = q; q = t; }
        if (q >= n) continue;  // the dummy column
        double* cp = A + static_cast<int64_t>(p) * m;
        double* cq = A + static_cast<int64_t>(q) * m;
        double g = 0.0;
        for (int64_t r = lane; r < m; r += 32) g += cp[r] * cq[r];
        g = warp_sum_d(g);
        const double alpha = norms[p], beta = norms[q];
        const double scale = sqrt(alpha * beta);
        if (scale <= 0.0 || fabs(g) <= tol * scale) continue;
        wl = fmax(wl, fabs(g) / scale);
        if (lane == 0) rotated = 1;
        const double zeta = (beta - alpha) / (2.0 * g);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        double np_ = 0.0, nq = 0.0;
        for (int64_t r = lane; r < m; r += 32) {
          const double x = cp[r], y = cq[r];
          const double xn = c * x - s * y, yn = s * x + c * y;
          cp[r] = xn;
          cq[r] = yn;
          np_ += xn * xn;
          nq += yn * yn;
        }
        np_ = warp_sum_d(np_);
        nq = warp_sum_d(nq);
        if (lane == 0) {
          norms[p] = np_;
          norms[q] = nq;
        }
      }
      __syncthreads();  // the next round pairs these columns with others
    }
    if (lane == 0) wmax[warp] = wl;
    __syncthreads();
    worst = 0.0;
    for (int w = 0; w < SV_WARPS; ++w) worst = fmax(worst, wmax[w]);
    const bool any = rotated != 0;
    __syncthreads();
    if (!any) {
      used = sweep + 1;
      break;
    }
  }
  // descending order: rank of each value (ties broken by index)
  for (int64_t i = threadIdx.x; i < n; i += SV_THREADS) {
    const double v = norms[i];
    int64_t rank = 0;
    for (int64_t j = 0; j < n; ++j) {
      const double u = norms[j];
      rank += (u > v) || (u == v && j < i);
    }
    sv[static_cast<int64_t>(blockIdx.x) * n + rank] = sqrt(fmax(v, 0.0));
  }
  if (threadIdx.x == 0) {
    if (resid) resid[blockIdx.x] = used > 0 ? 0.0 : worst;
    if (sweeps) sweeps[blockIdx.x] = used;
  }
}

}  // namespace
}  // namespace poetx

using namespace poetx;

extern "C" {

size_t poetx_singular_values_workspace_bytes(int64_t batch, int64_t rows, int64_t cols) {
  if (batch <= 0 || rows <= 0 || cols <= 0) return 256;
  return static_cast<size_t>(batch * rows * cols) * sizeof(double) + 256;
}

int poetx_singular_values(int64_t batch, int64_t rows, int64_t cols, const double* a, double* sv, double tol,
                          int max_sweeps, double* residual, int* sweeps, void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(batch >= 0 && rows >= 0 && cols >= 0, POETX_ESHAPE, "singular_values: negative shape");
  const int64_t n = rows < cols ? rows : cols, m = rows < cols ? cols : rows;
  POETX_REQUIRE(n <= SV_MAX_COLS, POETX_ESHAPE, "singular_values: min(rows, cols) = %lld > %lld",
                (long long)n, (long long)SV_MAX_COLS);
  POETX_REQUIRE(max_sweeps >= 1 && tol >= 0.0, POETX_ECONFIG, "singular_values: max_sweeps >= 1, tol >= 0");
  if (batch == 0 || n == 0) return POETX_OK;
  POETX_REQUIRE(a && sv && ws && ws_bytes >= poetx_singular_values_workspace_bytes(batch, rows, cols), POETX_ESHAPE,
                "singular_values: workspace too small");
  cudaStream_t st = as_stream(stream);
  double* w = static_cast<double*>(ws);
  const int64_t total = batch * rows * cols;
  const unsigned pg = static_cast<unsigned>(total / 256 + 1 < 148 * 16 ? total / 256 + 1 : 148 * 16);
  sv_prep_kernel<<<pg, 256, 0, st>>>(batch, rows, cols, a, w);
  POETX_LAUNCHED("sv_prep");
  jacobi_sv_kernel<<<static_cast<unsigned>(batch), SV_THREADS, static_cast<size_t>(n) * sizeof(double), st>>>(
      m, n, w, tol, max_sweeps, sv, residual, sweeps);
  POETX_LAUNCHED("jacobi_sv");
  return POETX_OK;
}

}  // extern "C"
