// PoetLinearLayer orchestration (layer.py:181-314) behind the C ABI:
// factors (CNP on both sides), forward chain, backward chain, merge.
// Kernels are stream-ordered; nothing here synchronises the host.
#include <cstdlib>

#include "common.cuh"
#include "simt_gemm.cuh"

namespace poetx {
int gemm(int dt, int out_dt, const GemmDesc& d, cudaStream_t st);
int gather2d(int dt, int64_t rows, int64_t cols, const int32_t* ridx, const int32_t* cidx,
             const void* x, void* y, cudaStream_t st);
int apply_features(int dt, int64_t T, int64_t nb, int64_t b, const void* g, int transpose,
                   const void* x, void* y, cudaStream_t st);
int apply_weight_rows(int dt, int64_t nb, int64_t b, int64_t cols, const void* g, int transpose,
                      const void* w, void* y, cudaStream_t st);
int apply_weight_rows_q8(int64_t nb, int64_t b, int64_t cols, const void* g, const int8_t* codes,
                         const float* scales, void* y, cudaStream_t st);
int apply_weight_cols_t_q8(int64_t m, int64_t nb, int64_t b, const void* g_p, const int8_t* codes,
                           const float* scales, void* y, cudaStream_t st);
int tc_matmul_q8(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA, const int8_t* B,
                 int64_t ldb, int transB, const float* scales, void* C, int64_t ldc, cudaStream_t st);
constexpr int kNotSupported = -100;  // POETX_ENOTSUPPORTED (tc_gemm.cuh)
int segmented_outer(int dt, int64_t T, int64_t nb, int64_t b, const void* x, const void* y,
                    void* out, int accumulate, Workspace& ws, cudaStream_t st);
size_t cnp_ws_bytes(int dt, int64_t nb, int64_t b, int k);
size_t outer_ws_bytes(int dt, int64_t T, int64_t nb, int64_t b);
size_t tc_outer_ws_bytes(int64_t T, int64_t nb, int64_t b);
int quant_dequant(int dt, int64_t rows, int64_t cols, const int8_t* codes, const void* scales,
                  const int32_t* ri, const int32_t* ci, void* out, cudaStream_t st, int64_t ld = 0);
int quant_rows(int dt, int64_t rows, int64_t cols, const void* w, int8_t* codes, void* scales, cudaStream_t st);
int quant_gather(int dt, int64_t rows, int64_t cols, const int32_t* ri, const int32_t* ci, const int8_t* codes,
                 const void* scales, int8_t* codes_out, void* scales_out, cudaStream_t st, int64_t ld = 0);
}  // namespace poetx

using namespace poetx;

namespace {

int check_desc(const poetx_layer_desc* d) {
  POETX_REQUIRE(d != nullptr, POETX_ESHAPE, "layer: null descriptor");
  POETX_REQUIRE(valid_dtype(d->dtype), POETX_ESHAPE, "layer: unsupported dtype %d", d->dtype);
  POETX_REQUIRE(d->b >= 1, POETX_ECONFIG, "block_size must be >= 1, got %lld", (long long)d->b);
  POETX_REQUIRE(d->m % d->b == 0 && d->n % d->b == 0, POETX_ECONFIG,
                "layer dims (%lld, %lld) must both be divisible by block_size %lld",
                (long long)d->m, (long long)d->n, (long long)d->b);
  POETX_REQUIRE(d->variant == POETX_FAST || d->variant == POETX_MEM, POETX_ECONFIG,
                "variant must be fast or mem");
  POETX_REQUIRE(d->neumann_k >= 1, POETX_ECONFIG, "neumann_k must be >= 1, got %d", d->neumann_k);
  POETX_REQUIRE(!d->pm_codes || d->variant == POETX_MEM, POETX_ECONFIG,
                "quantized base requires the mem variant");
  POETX_REQUIRE(!d->pm_codes || d->pm_scales, POETX_ESHAPE, "layer: quantized base without scales");
  return POETX_OK;
}

bool quantized(const poetx_layer_desc* d) { return d->pm_codes != nullptr; }

// BF16 layers reassociate the products around the frozen weight so the
// block-diagonal factors are applied to the WEIGHT (m x n) instead of the
// activations (T x m, T x n):
//   forward   t  = (u bd(G_R)) PM      = u  (bd(G_R) PM)      W2 = G_R PM
//   backward  da = (dv bd(G_P)^T) PM^T = dv (PM bd(G_P))^T    W1 = PM G_P
// one weight-sized pass per product instead of a token-sized one (1.5-4x
// fewer bytes at T = 8192); the result is rounded to bf16 once either way.
bool reassoc(const poetx_layer_desc* d) {
  static int on = [] {
    const char* e = getenv("POETX_REASSOC");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on && d->fold_weight && d->dtype == POETX_BF16 && d->b % 64 == 0 && d->b <= 256 && d->n % 256 == 0;
}

// POET-XQ: scratch for the dequantized premerged weight, reserved up front
// in the call's workspace (so the layout never depends on which products end
// up needing it); nullptr for a float base
int reserve_deq(const poetx_layer_desc* d, Workspace& w, void*& out) {
  out = nullptr;
  if (!quantized(d)) return POETX_OK;
  out = w.take_bytes(static_cast<size_t>(d->m * d->n) * elt_size(d->dtype));
  POETX_REQUIRE(out, POETX_ESHAPE, "layer: workspace too small for the dequantized weight");
  return POETX_OK;
}

// POET-XQ products that take the int8 codes straight into the pair GEMM's
// producer (dequantized on chip, bit-identical to the dequantizer + bf16
// GEMM): mm2, the adjoint and the W2 = bd(G_R) PM fold.  Only products that
// cannot (W1 = PM bd(G_P), non-pair shapes) dequantize PM into workspace
// scratch -- lazily, once per call.  POETX_Q8_GEMM=0: always dequantize,
// =1: folds only (A/B).
bool q8_gemm(const poetx_layer_desc* d) {
  static int on = [] {
    const char* e = getenv("POETX_Q8_GEMM");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on && quantized(d) && d->dtype == POETX_BF16 && d->n % 16 == 0;
}
// the main products (mm2 / adjoint) take codes too unless POETX_Q8_GEMM=1
// (folds only; tools/q8bench.py: at or below dequantize + GEMM at the
// Llama-8B shapes, within 5% at the 1B ones)
bool q8_main() {
  static int on = [] {
    const char* e = getenv("POETX_Q8_GEMM");
    return e && e[0] == '1' ? 0 : 1;
  }();
  return on != 0;
}
// the backward weight fold W1 of a POET-XQ layer is built as W1^T straight
// from the codes (pair GEMM, b = 256, m % 256 == 0); the adjoint reads it
// as its K x N operand
bool w1_transposed(const poetx_layer_desc* d) {
  return q8_gemm(d) && d->b == 256 && d->m % 256 == 0;
}
struct PmSource {
  const poetx_layer_desc* d;
  void* scratch;  // reserve_deq
  cudaStream_t st;
  bool filled = false;
  // the bf16 (or fp32/fp64) premerged weight; POET-XQ codes dequantized into
  // the scratch on first use (the device analogue of quant.py's dequantizer)
  int get(const void*& out) {
    if (!quantized(d)) {
      out = d->premerged;
      return POETX_OK;
    }
    if (!filled) {
      POETX_TRY(quant_dequant(d->dtype, d->m, d->n, d->pm_codes, d->pm_scales, nullptr, nullptr, scratch, st));
      filled = true;
    }
    out = scratch;
    return POETX_OK;
  }
  // c[T, N] = a[T, K] . PM (transB 0: PM is [K, N]) or a . PM^T (transB 1: PM is [N, K])
  int matmul(int64_t T, int64_t N, int64_t K, const void* a, int transB, void* c) {
    if (q8_gemm(d) && q8_main()) {
      int rc = tc_matmul_q8(T, N, K, a, K, 0, d->pm_codes, d->n, transB, static_cast<const float*>(d->pm_scales), c,
                            N, st);
      if (rc != kNotSupported) return rc;
    }
    const void* pm;
    POETX_TRY(get(pm));
    return poetx_matmul(d->dtype, T, N, K, a, K, 0, pm, d->n, transB, c, N, 0, st);
  }
  // W2 = bd(G_R) PM
  int fold_in(const void* g_r, void* out) {
    if (q8_gemm(d)) {
      int rc = apply_weight_rows_q8(d->m / d->b, d->b, d->n, g_r, d->pm_codes, static_cast<const float*>(d->pm_scales),
                                    out, st);
      if (rc != kNotSupported) return rc;
    }
    const void* pm;
    POETX_TRY(get(pm));
    return apply_weight_rows(d->dtype, d->m / d->b, d->b, d->n, g_r, 0, pm, out, st);
  }
  // W1 = PM bd(G_P) -- stored TRANSPOSED ([n, m]) for POET-XQ layers that
  // take codes (w1_transposed), so its producer can read the codes
  int fold_out(const void* g_p, void* out) {
    if (w1_transposed(d)) {
      int rc = apply_weight_cols_t_q8(d->m, d->n / d->b, d->b, g_p, d->pm_codes,
                                      static_cast<const float*>(d->pm_scales), out, st);
      if (rc != kNotSupported) return rc;
      set_error("layer: transposed int8 fold unsupported for this shape");
      return POETX_ESHAPE;
    }
    const void* pm;
    POETX_TRY(get(pm));
    return apply_features(d->dtype, d->m, d->n / d->b, d->b, g_p, 0, pm, out, st);
  }
};

// BF16 layers with k = 3, b in {128, 256} and NO Q^2 cache in the factor
// struct run the CNP as the fused tensor-core kernels (csrc/cnp_fused.cu);
// a supplied Q^2 cache selects the CUDA-core fp32 path (merge accuracy)
bool cnp_fused_ok(const poetx_layer_desc* d, const poetx_layer_factors_t* f) {
  return d->dtype == POETX_BF16 && d->neumann_k == 3 && !f->q2_r && !f->q2_p && poetx_cnp_fused_supported(d->b);
}

// BF16 layers with b in {128, 256} merge on tensor cores (csrc/merge_tc.cu);
// POETX_MERGE_TC=0 keeps the CUDA-core fp32 passes (A/B timing)
bool merge_tc_ok(const poetx_layer_desc* d) {
  static int on = [] {
    const char* e = getenv("POETX_MERGE_TC");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on && d->dtype == POETX_BF16 && poetx_merge_tc_supported(d->b) && d->n % 8 == 0;
}

// G used by the activation path: the bf16 copy for BF16 layers
const void* act_g(const poetx_layer_desc* d, const void* g, const void* g16) {
  return d->dtype == POETX_BF16 ? g16 : g;
}

size_t cnp_bwd_ws(const poetx_layer_desc* d) {
  int pdt = param_dtype(d->dtype);
  size_t r = cnp_ws_bytes(pdt, d->m / d->b, d->b, d->neumann_k);
  size_t p = cnp_ws_bytes(pdt, d->n / d->b, d->b, d->neumann_k);
  return r > p ? r : p;
}

template <typename Tin, typename Tout>
__global__ void gather_convert_kernel(int64_t rows, int64_t cols, const int32_t* __restrict__ ridx,
                                      const int32_t* __restrict__ cidx, const Tin* __restrict__ x,
                                      Tout* __restrict__ y) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const Tin* xr = x + static_cast<int64_t>(ridx ? ridx[r] : r) * cols;
    Tout* yr = y + r * cols;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
      yr[j] = cvt<Tin, Tout>(xr[cidx ? cidx[j] : j]);
  }
}

__global__ void compose_kernel(int64_t n, const int32_t* __restrict__ inv_old,
                               const int32_t* __restrict__ fwd_new, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = inv_old[fwd_new[i]];
}

template <typename Tin, typename Tout>
int gather_convert(int64_t rows, int64_t cols, const int32_t* ridx, const int32_t* cidx,
                   const void* x, void* y, cudaStream_t st) {
  unsigned grid = static_cast<unsigned>(rows < 148 * 16 ? rows : 148 * 16);
  gather_convert_kernel<Tin, Tout><<<grid, 256, 0, st>>>(rows, cols, ridx, cidx,
                                                         static_cast<const Tin*>(x),
                                                         static_cast<Tout*>(y));
  POETX_LAUNCHED("gather_convert");
  return POETX_OK;
}

int gather_to(int src_dt, int dst_dt, int64_t rows, int64_t cols, const int32_t* ridx,
              const int32_t* cidx, const void* x, void* y, cudaStream_t st) {
  if (src_dt == dst_dt) return gather2d(src_dt, rows, cols, ridx, cidx, x, y, st);
  if (src_dt == POETX_F32 && dst_dt == POETX_BF16)
    return gather_convert<float, __nv_bfloat16>(rows, cols, ridx, cidx, x, y, st);
  if (src_dt == POETX_BF16 && dst_dt == POETX_F32)
    return gather_convert<__nv_bfloat16, float>(rows, cols, ridx, cidx, x, y, st);
  set_error("gather_to: unsupported conversion %d -> %d", src_dt, dst_dt);
  return POETX_ESHAPE;
}

// The backward's two segmented outer products (dG_P = t^T dv, dG_R = u^T da)
// only READ buffers the main chain (dt -> adjoint GEMM -> du) reads too, so
// they fork onto the caller-owned desc->side_stream with events and join at
// the end: they fill the SMs the main chain's kernel tails leave idle.
// Inside a CUDA-graph capture the fork/join become graph edges.  The events
// live for one call; the library keeps no stream or event of its own.
bool side_enabled() {
  static int on = [] {
    const char* e = getenv("POETX_LAYER_SIDE");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on != 0;
}
struct Side {
  cudaStream_t s = nullptr;
  cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
  explicit Side(void* stream) {
    if (!stream) return;
    for (auto& ev : e) {
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        release();
        return;
      }
    }
    s = as_stream(stream);
  }
  void release() {
    for (auto& ev : e) {
      if (ev) cudaEventDestroy(ev);  // deferred by the driver until the event completes
      ev = nullptr;
    }
    s = nullptr;
  }
  ~Side() { release(); }
};

}  // namespace

extern "C" {

size_t poetx_layer_workspace_bytes(const poetx_layer_desc* d, int64_t T) {
  if (check_desc(d) != POETX_OK) return 0;
  const size_t e = elt_size(d->dtype), acc = elt_size(param_dtype(d->dtype));
  const int64_t w = d->m > d->n ? d->m : d->n;
  size_t act = align_up(static_cast<size_t>(T) * w * e);
  size_t grads = align_up(static_cast<size_t>(d->m * d->b) * acc) +
                 align_up(static_cast<size_t>(d->n * d->b) * acc);
  size_t outer = outer_ws_bytes(d->dtype, T, d->m / d->b, d->b);
  size_t outer2 = outer_ws_bytes(d->dtype, T, d->n / d->b, d->b);
  if (outer2 > outer) outer = outer2;
  if (d->dtype == POETX_BF16) {
    size_t t1 = tc_outer_ws_bytes(T, d->m / d->b, d->b), t2 = tc_outer_ws_bytes(T, d->n / d->b, d->b);
    if (t1 > outer) outer = t1;
    if (t2 > outer) outer = t2;
  }
  size_t cnp = cnp_bwd_ws(d);
  const size_t deq = quantized(d) ? align_up(static_cast<size_t>(d->m * d->n) * e) : 0;
  const size_t wfold = reassoc(d) ? 2 * align_up(static_cast<size_t>(d->m * d->n) * e) : 0;
  return 4 * act + grads + deq + wfold + (outer > cnp ? outer : cnp) + 8192;
}

int poetx_layer_factors(const poetx_layer_desc* d, poetx_layer_factors_t* f, void* ws,
                        size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(f && f->packed_r && f->packed_p && f->g_r && f->g_p, POETX_ESHAPE,
                "layer_factors: missing factor buffers");
  if (d->dtype == POETX_BF16)
    POETX_REQUIRE(f->g_r_lowp && f->g_p_lowp, POETX_ESHAPE, "layer_factors: bf16 layer needs lowp G");
  const int pdt = param_dtype(d->dtype);
  const int k = d->neumann_k;
  if (cnp_fused_ok(d, f)) {
    POETX_TRY(poetx_cnp_forward_fused(d->m / d->b, d->b, static_cast<const float*>(f->packed_r), f->g_r_lowp,
                                      static_cast<float*>(f->g_r), stream));
    return poetx_cnp_forward_fused(d->n / d->b, d->b, static_cast<const float*>(f->packed_p), f->g_p_lowp,
                                   static_cast<float*>(f->g_p), stream);
  }
  void* q2r = k == 3 ? f->q2_r : nullptr;
  void* q2p = k == 3 ? f->q2_p : nullptr;
  POETX_TRY(poetx_cnp_forward(pdt, d->m / d->b, d->b, k, nullptr, f->packed_r, f->g_r,
                              d->dtype == POETX_BF16 ? f->g_r_lowp : nullptr, q2r, ws, ws_bytes,
                              stream));
  POETX_TRY(poetx_cnp_forward(pdt, d->n / d->b, d->b, k, nullptr, f->packed_p, f->g_p,
                              d->dtype == POETX_BF16 ? f->g_p_lowp : nullptr, q2p, ws, ws_bytes,
                              stream));
  return POETX_OK;
}

int poetx_layer_forward_ex(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                           const void* x, void* z, void* saved_t, int flags, void* ws,
                           size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(T >= 0 && x && z && f, POETX_ESHAPE, "layer_forward: bad arguments");
  if (T == 0) return POETX_OK;
  cudaStream_t st = as_stream(stream);
  const int dt = d->dtype;
  const int64_t w = d->m > d->n ? d->m : d->n;
  const size_t e = elt_size(dt);
  const bool in_gathered = flags & POETX_IN_GATHERED, out_raw = flags & POETX_OUT_UNSCATTERED;
  Workspace wsp(ws, ws_bytes);
  void* b1 = wsp.take_bytes(T * w * e);
  void* b2 = wsp.take_bytes(T * w * e);
  void* b3 = wsp.take_bytes(T * w * e);
  POETX_REQUIRE(b1 && b2 && b3, POETX_ESHAPE, "layer_forward: workspace too small");
  void* deq;
  POETX_TRY(reserve_deq(d, wsp, deq));
  PmSource pm{d, deq, st};
  void* t = saved_t ? saved_t : b3;
  // u = x[:, pi_in]  (permute_features 'inverse', layer.py:220) -- or supplied
  const void* u = x;
  if (!in_gathered) {
    POETX_TRY(gather2d(dt, T, d->m, nullptr, d->perm_in_fwd, x, b1, st));
    u = b1;
  }
  if (reassoc(d)) {
    // t = u (bd(G_R) PM)  (mm1 folded into the weight, layer.py:221-222)
    const void* w2 = f->w_in_fold;
    if (!w2) {
      void* w = wsp.take_bytes(d->m * d->n * e);
      POETX_REQUIRE(w, POETX_ESHAPE, "layer_forward: workspace too small");
      POETX_TRY(pm.fold_in(act_g(d, f->g_r, f->g_r_lowp), w));
      w2 = w;
    }
    POETX_TRY(poetx_matmul(dt, T, d->n, d->m, u, d->m, 0, w2, d->n, 0, t, d->n, 0, stream));
  } else {
    // a = u blockdiag(G_R)  (mm1, layer.py:221)
    POETX_TRY(apply_features(dt, T, d->m / d->b, d->b, act_g(d, f->g_r, f->g_r_lowp), 0, u, b2, st));
    // t = a PM  (mm2, layer.py:222)
    POETX_TRY(pm.matmul(T, d->n, d->m, b2, 0, t));
  }
  // v = t blockdiag(G_P)  (mm3, layer.py:223)
  void* v = out_raw ? z : b1;
  POETX_TRY(apply_features(dt, T, d->n / d->b, d->b, act_g(d, f->g_p, f->g_p_lowp), 0, t, v, st));
  // z = v[:, pi_out^-1]  (permute_features 'forward', layer.py:224) -- or left to the caller
  if (!out_raw) POETX_TRY(gather2d(dt, T, d->n, nullptr, d->perm_out_inv, b1, z, st));
  return POETX_OK;
}

int poetx_layer_forward(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                        const void* x, void* z, void* saved_t, void* ws, size_t ws_bytes,
                        void* stream) {
  return poetx_layer_forward_ex(d, f, T, x, z, saved_t, 0, ws, ws_bytes, stream);
}

static int layer_backward_impl(const poetx_layer_desc* d, const poetx_layer_factors_t* f,
                               int64_t T, const void* x, const void* dz, const void* saved_t,
                               void* dx, void* dpacked_r, void* dpacked_p, void* dg_r_out,
                               void* dg_p_out, int accumulate, int flags, void* ws, size_t ws_bytes,
                               void* stream) {
  cudaStream_t st = as_stream(stream);
  const int dt = d->dtype, pdt = param_dtype(dt);
  const int64_t w = d->m > d->n ? d->m : d->n, b = d->b, nbr = d->m / b, nbp = d->n / b;
  const size_t e = elt_size(dt), acc = elt_size(pdt);
  const bool dg_mode = dg_r_out != nullptr;
  Workspace wsp(ws, ws_bytes);
  void* b1 = wsp.take_bytes(T * w * e);
  void* b2 = wsp.take_bytes(T * w * e);
  void* b3 = wsp.take_bytes(T * w * e);
  void* b4 = wsp.take_bytes(T * w * e);
  void* dgr = dg_mode ? dg_r_out : wsp.take_bytes(nbr * b * b * acc);
  void* dgp = dg_mode ? dg_p_out : wsp.take_bytes(nbp * b * b * acc);
  POETX_REQUIRE(b1 && b2 && b3 && b4 && dgr && dgp, POETX_ESHAPE,
                "layer_backward: workspace too small");
  void* deq;
  POETX_TRY(reserve_deq(d, wsp, deq));
  PmSource pm{d, deq, st};
  const int dg_acc = dg_mode ? accumulate : 0;
  const void* gr = act_g(d, f->g_r, f->g_r_lowp);
  const void* gp = act_g(d, f->g_p, f->g_p_lowp);
  const bool in_gathered = flags & POETX_IN_GATHERED, dz_gathered = flags & POETX_DZ_GATHERED;
  const bool dx_raw = flags & POETX_DX_UNSCATTERED;
  // dv = dz[:, pi_out]  (layer.py:238) -- or supplied
  const void* dv = dz;
  if (!dz_gathered) {
    POETX_TRY(gather2d(dt, T, d->n, nullptr, d->perm_out_fwd, dz, b1, st));
    dv = b1;
  }
  const bool ra = reassoc(d);
  const bool own_w1 = ra && !f->w_out_fold, own_w2 = ra && !saved_t && !f->w_in_fold;
  void* w1 = own_w1 ? wsp.take_bytes(d->m * d->n * e) : nullptr;  // PM bd(G_P)
  void* w2 = own_w2 ? wsp.take_bytes(d->m * d->n * e) : nullptr;  // bd(G_R) PM
  POETX_REQUIRE((!own_w1 || w1) && (!own_w2 || w2), POETX_ESHAPE, "layer_backward: workspace too small");
  Workspace tail(static_cast<char*>(ws) + wsp.used, ws_bytes - wsp.used);
  const void* t = saved_t;
  if (!t) {
    // mem variant: recompute u, a, t with the forward's kernels (bitwise equal)
    const void* u0 = x;
    if (!in_gathered) {
      POETX_TRY(gather2d(dt, T, d->m, nullptr, d->perm_in_fwd, x, b2, st));
      u0 = b2;
    }
    if (ra) {
      if (own_w2) POETX_TRY(pm.fold_in(gr, w2));
      const void* wi = own_w2 ? w2 : f->w_in_fold;
      POETX_TRY(poetx_matmul(dt, T, d->n, d->m, u0, d->m, 0, wi, d->n, 0, b4, d->n, 0, stream));
    } else {
      POETX_TRY(apply_features(dt, T, nbr, b, gr, 0, u0, b3, st));
      POETX_TRY(pm.matmul(T, d->n, d->m, b3, 0, b4));
    }
    t = b4;
  }
  // the two segmented outer products run on a side stream unless the main
  // chain would overwrite dv's buffer with u (b1) while the first one reads it
  Side side((side_enabled() && (dz_gathered || in_gathered)) ? d->side_stream : nullptr);
  Side* sd = side.s ? &side : nullptr;
  cudaStream_t so = sd ? sd->s : st;
  if (sd) {
    cudaEventRecord(sd->e[0], st);
    cudaStreamWaitEvent(so, sd->e[0], 0);
  }
  // dG_P = segmented_outer(t, dv)  (layer.py:247)
  POETX_TRY(segmented_outer(dt, T, nbp, b, t, dv, dgp, dg_acc, tail, so));
  if (ra) {
    // da = dv (PM bd(G_P))^T  (layer.py:248-249 with dt folded into the weight)
    if (own_w1) POETX_TRY(pm.fold_out(gp, w1));
    const void* wo = own_w1 ? w1 : f->w_out_fold;
    if (w1_transposed(d))  // W1^T [n, m] is the K x N operand
      POETX_TRY(poetx_matmul(dt, T, d->m, d->n, dv, d->n, 0, wo, d->m, 0, b3, d->m, 0, stream));
    else
      POETX_TRY(poetx_matmul(dt, T, d->m, d->n, dv, d->n, 0, wo, d->n, 1, b3, d->m, 0, stream));
  } else {
    // dt = dv blockdiag(G_P)^T  (layer.py:248)
    POETX_TRY(apply_features(dt, T, nbp, b, gp, 1, dv, b2, st));
    // da = dt PM^T  (layer.py:249)
    POETX_TRY(pm.matmul(T, d->m, d->n, b2, 1, b3));
  }
  // u = x[:, pi_in]  (layer.py:250) -- or the supplied pre-gathered input
  const void* u = x;
  if (!in_gathered) {
    POETX_TRY(gather2d(dt, T, d->m, nullptr, d->perm_in_fwd, x, b1, st));
    u = b1;
  }
  // dG_R = segmented_outer(u, da)  (layer.py:251)
  Workspace tail2(static_cast<char*>(ws) + wsp.used, ws_bytes - wsp.used);
  if (sd) {
    cudaEventRecord(sd->e[1], st);
    cudaStreamWaitEvent(so, sd->e[1], 0);
  }
  POETX_TRY(segmented_outer(dt, T, nbr, b, u, b3, dgr, dg_acc, tail2, so));
  if (dx) {
    // du = da blockdiag(G_R)^T ; dx = du[:, pi_in^-1]  (layer.py:252-253)
    if (dx_raw) {
      POETX_TRY(apply_features(dt, T, nbr, b, gr, 1, b3, dx, st));
    } else {
      POETX_TRY(apply_features(dt, T, nbr, b, gr, 1, b3, b2, st));
      POETX_TRY(gather2d(dt, T, d->m, nullptr, d->perm_in_inv, b2, dx, st));
    }
  }
  if (sd) {  // join: everything after this call sees dG_R / dG_P
    cudaEventRecord(sd->e[2], so);
    cudaStreamWaitEvent(st, sd->e[2], 0);
  }
  if (dg_mode) return POETX_OK;
  // packed grads = P(cnp_backward(.))  (layer.py:254-255)
  void* cws = static_cast<char*>(ws) + wsp.used;
  size_t cwsb = ws_bytes - wsp.used;
  const int k = d->neumann_k;
  if (cnp_fused_ok(d, f)) {
    // BF16 layer without a Q^2 cache: the fused tensor-core CNP backward
    // recomputes Q^2 on chip and writes the packed gradients (cnp_fused.cu)
    POETX_TRY(poetx_cnp_backward_fused(nbr, b, static_cast<const float*>(f->packed_r),
                                       static_cast<const float*>(dgr), static_cast<float*>(dpacked_r), accumulate,
                                       stream));
    return poetx_cnp_backward_fused(nbp, b, static_cast<const float*>(f->packed_p), static_cast<const float*>(dgp),
                                    static_cast<float*>(dpacked_p), accumulate, stream);
  }
  POETX_TRY(poetx_cnp_backward(pdt, nbr, b, k, nullptr, f->packed_r, k == 3 ? f->q2_r : nullptr,
                               dgr, nullptr, dpacked_r, accumulate, cws, cwsb, stream));
  POETX_TRY(poetx_cnp_backward(pdt, nbp, b, k, nullptr, f->packed_p, k == 3 ? f->q2_p : nullptr,
                               dgp, nullptr, dpacked_p, accumulate, cws, cwsb, stream));
  return POETX_OK;
}

int poetx_layer_backward(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                         const void* x, const void* dz, const void* saved_t, void* dx,
                         void* dpacked_r, void* dpacked_p, int accumulate, void* ws,
                         size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(T >= 0 && x && dz && f && dpacked_r && dpacked_p, POETX_ESHAPE,
                "layer_backward: bad arguments");
  return layer_backward_impl(d, f, T, x, dz, saved_t, dx, dpacked_r, dpacked_p, nullptr, nullptr,
                             accumulate, 0, ws, ws_bytes, stream);
}

int poetx_layer_backward_dg(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                            const void* x, const void* dz, const void* saved_t, void* dx,
                            void* dg_r, void* dg_p, int accumulate, int flags, void* ws,
                            size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(T >= 0 && x && dz && f && dg_r && dg_p, POETX_ESHAPE,
                "layer_backward_dg: bad arguments");
  return layer_backward_impl(d, f, T, x, dz, saved_t, dx, nullptr, nullptr, dg_r, dg_p,
                             accumulate, flags, ws, ws_bytes, stream);
}

int poetx_layer_weight_fold(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int which, void* out,
                            void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(d->dtype == POETX_BF16 && f && out && (which == 0 || which == 1), POETX_ESHAPE,
                "layer_weight_fold: BF16 layer, factors and output required");
  POETX_REQUIRE(f->g_r_lowp && f->g_p_lowp, POETX_ESHAPE, "layer_weight_fold: bf16 factors required");
  cudaStream_t st = as_stream(stream);
  Workspace wsp(ws, ws_bytes);
  void* deq;
  POETX_TRY(reserve_deq(d, wsp, deq));
  PmSource pm{d, deq, st};
  return which == 0 ? pm.fold_in(f->g_r_lowp, out) : pm.fold_out(f->g_p_lowp, out);
}

size_t poetx_merge_workspace_bytes(const poetx_layer_desc* d) {
  if (check_desc(d) != POETX_OK) return 0;
  size_t acc = elt_size(param_dtype(d->dtype));
  size_t q = quantized(d) ? align_up(static_cast<size_t>(d->m * d->n)) + align_up(static_cast<size_t>(d->m) * acc) : 0;
  return 3 * align_up(static_cast<size_t>(d->m * d->n) * acc) +
         align_up(static_cast<size_t>(d->m + d->n) * 4) + q + 4096;
}

int poetx_layer_merge(const poetx_layer_desc* d, const void* g_r, const void* g_p,
                      const int32_t* new_in_fwd, const int32_t* new_out_fwd, void* premerged_out,
                      void* w_out, void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(g_r && g_p, POETX_ESHAPE, "layer_merge: missing factors");
  cudaStream_t st = as_stream(stream);
  const int dt = d->dtype, pdt = param_dtype(dt);
  const int64_t m = d->m, n = d->n, b = d->b;
  const size_t acc = elt_size(pdt);
  Workspace wsp(ws, ws_bytes);
  void* pm = wsp.take_bytes(m * n * acc);
  void* mid1 = wsp.take_bytes(m * n * acc);
  void* mid2 = wsp.take_bytes(m * n * acc);
  int32_t* ridx = wsp.take<int32_t>(m);
  int32_t* cidx = wsp.take<int32_t>(n);
  POETX_REQUIRE(pm && mid1 && mid2 && ridx && cidx, POETX_ESHAPE, "layer_merge: workspace too small");
  // BF16 layers, b in {128, 256}: mid = blockdiag(G_R) PM blockdiag(G_P) as
  // ONE tensor-core pass (csrc/merge_tc.cu: fp32 factors split hi/lo, fp32
  // accumulation), bf16 out, then the composite re-permutation gather
  if (merge_tc_ok(d)) {
    POETX_TRY(poetx_merge_tc(m, n, b, static_cast<const float*>(g_r), static_cast<const float*>(g_p),
                             quantized(d) ? nullptr : d->premerged, d->pm_codes,
                             static_cast<const float*>(d->pm_scales), n, mid2, POETX_BF16, n, stream));
    if (w_out) POETX_TRY(gather2d(dt, m, n, d->perm_in_inv, d->perm_out_inv, mid2, w_out, st));
    if (premerged_out) {
      POETX_REQUIRE(new_in_fwd && new_out_fwd, POETX_ESHAPE, "layer_merge: missing new permutations");
      compose_kernel<<<grid_for(m, 256), 256, 0, st>>>(m, d->perm_in_inv, new_in_fwd, ridx);
      POETX_LAUNCHED("compose");
      compose_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, d->perm_out_inv, new_out_fwd, cidx);
      POETX_LAUNCHED("compose");
      POETX_TRY(gather2d(dt, m, n, ridx, cidx, mid2, premerged_out, st));
    }
    return POETX_OK;
  }
  // mid = blockdiag(G_R) PM blockdiag(G_P) in the parameter type (layer.py:269-271)
  const void* pm_src = d->premerged;
  if (quantized(d)) {
    POETX_TRY(quant_dequant(pdt, m, n, d->pm_codes, d->pm_scales, nullptr, nullptr, pm, st));
    pm_src = pm;
  } else if (dt == POETX_BF16) {
    POETX_TRY(gather_to(POETX_BF16, POETX_F32, m, n, nullptr, nullptr, d->premerged, pm, st));
    pm_src = pm;
  }
  POETX_TRY(apply_weight_rows(pdt, m / b, b, n, g_r, 0, pm_src, mid1, st));
  POETX_TRY(apply_features(pdt, m, n / b, b, g_p, 0, mid1, mid2, st));
  if (w_out) {
    // W = Psi_m^T mid Psi_n : W[r, c] = mid[inv_in(r), inv_out(c)]  (layer.py:272-273)
    POETX_TRY(gather_to(pdt, dt, m, n, d->perm_in_inv, d->perm_out_inv, mid2, w_out, st));
  }
  if (premerged_out) {
    POETX_REQUIRE(new_in_fwd && new_out_fwd, POETX_ESHAPE, "layer_merge: missing new permutations");
    // PM'[i, j] = W[new_in(i), new_out(j)] = mid[inv_in(new_in(i)), inv_out(new_out(j))]
    compose_kernel<<<grid_for(m, 256), 256, 0, st>>>(m, d->perm_in_inv, new_in_fwd, ridx);
    POETX_LAUNCHED("compose");
    compose_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, d->perm_out_inv, new_out_fwd, cidx);
    POETX_LAUNCHED("compose");
    POETX_TRY(gather_to(pdt, dt, m, n, ridx, cidx, mid2, premerged_out, st));
  }
  return POETX_OK;
}

int poetx_layer_merge_quant(const poetx_layer_desc* d, const void* g_r, const void* g_p,
                            const int32_t* new_in_fwd, const int32_t* new_out_fwd, int8_t* codes_out,
                            void* scales_out, void* w_out, void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check_desc(d));
  POETX_REQUIRE(quantized(d), POETX_ESTATE, "layer_merge_quant: layer base is not quantized");
  POETX_REQUIRE(g_r && g_p && new_in_fwd && new_out_fwd && codes_out && scales_out, POETX_ESHAPE,
                "layer_merge_quant: missing arguments");
  cudaStream_t st = as_stream(stream);
  const int dt = d->dtype, pdt = param_dtype(dt);
  const int64_t m = d->m, n = d->n, b = d->b;
  const size_t acc = elt_size(pdt);
  Workspace wsp(ws, ws_bytes);
  void* pm = wsp.take_bytes(m * n * acc);
  void* mid1 = wsp.take_bytes(m * n * acc);
  void* mid2 = wsp.take_bytes(m * n * acc);
  int32_t* ridx = wsp.take<int32_t>(m);
  int32_t* cidx = wsp.take<int32_t>(n);
  int8_t* qc = wsp.take<int8_t>(static_cast<size_t>(m * n));
  void* qs = wsp.take_bytes(m * acc);
  POETX_REQUIRE(pm && mid1 && mid2 && ridx && cidx && qc && qs, POETX_ESHAPE, "layer_merge_quant: workspace too small");
  // mid = blockdiag(G_R) deq(PM) blockdiag(G_P)  (layer.py:260-271, dequantized premerged);
  // on tensor cores the row scales fold into G_R's columns and the codes are
  // exact bf16 operands (csrc/merge_tc.cu), fp32 out for the requantization
  if (merge_tc_ok(d)) {
    POETX_TRY(poetx_merge_tc(m, n, b, static_cast<const float*>(g_r), static_cast<const float*>(g_p), nullptr,
                             d->pm_codes, static_cast<const float*>(d->pm_scales), n, mid2, POETX_F32, n, stream));
  } else {
    POETX_TRY(quant_dequant(pdt, m, n, d->pm_codes, d->pm_scales, nullptr, nullptr, pm, st));
    POETX_TRY(apply_weight_rows(pdt, m / b, b, n, g_r, 0, pm, mid1, st));
    POETX_TRY(apply_features(pdt, m, n / b, b, g_p, 0, mid1, mid2, st));
  }
  if (w_out) POETX_TRY(gather_to(pdt, dt, m, n, d->perm_in_inv, d->perm_out_inv, mid2, w_out, st));
  // requantize per row (rows of the new base W are rows of mid, columns only
  // permuted: absmax and every code are invariant), then gather the codes
  // into the new premerged order PM'[i,j] = W[new_in(i), new_out(j)]
  POETX_TRY(quant_rows(pdt, m, n, mid2, qc, qs, st));
  compose_kernel<<<grid_for(m, 256), 256, 0, st>>>(m, d->perm_in_inv, new_in_fwd, ridx);
  POETX_LAUNCHED("compose");
  compose_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, d->perm_out_inv, new_out_fwd, cidx);
  POETX_LAUNCHED("compose");
  return quant_gather(dt, m, n, ridx, cidx, qc, qs, codes_out, scales_out, st);
}

}  // extern "C"
