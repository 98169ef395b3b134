// Row-staged BF16 kernels that fuse the POET-X layer's feature
// permutations (permute.py:95-110: u = x[:, pi_in], z = v[:, pi_out^-1])
// into the elementwise neighbours a decoder block needs anyway, so no
// standalone permutation pass touches HBM:
//
//   rmsnorm_gather      y = rmsnorm(x) * w ; u_k = y[:, idx_k]   (k <= 3 consumers)
//   rmsnorm_gather_bwd  dy = sum_k du_k[:, inv_k] ; RMSNorm backward ; dw partials
//   swiglu_gather       u_down[:, j] = silu(v_g[:, cg[j]]) * v_u[:, cu[j]]
//                       (cg = inv_g o fwd_down, cu = inv_u o fwd_down: two
//                       output scatters and one input gather in one index map)
//   swiglu_gather_bwd   dv_g, dv_u through the composed maps
//   rope_scatter        out = RoPE(v[:, inv])   and its backward
//   scatter_add         out = h + v[:, inv]     (residual)
//
// One CTA per row (grid-stride), the row(s) staged in shared memory with
// 16-byte coalesced loads, outputs written with 16-byte coalesced stores.
#include "common.cuh"

namespace poetx {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 3;

struct IdxList {
  const int32_t* idx[kMaxK];
  void* ptr[kMaxK];
};

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.f;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ void load_row(__nv_bfloat16* s, const __nv_bfloat16* g, int64_t n) {
  const uint4* src = reinterpret_cast<const uint4*>(g);
  uint4* dst = reinterpret_cast<uint4*>(s);
  for (int64_t i = threadIdx.x; i < n / 8; i += blockDim.x) dst[i] = __ldcs(src + i);
}

// gather 8 consecutive outputs j0..j0+7 from a staged row through idx
template <typename F>
__device__ __forceinline__ uint4 gather8(const int32_t* idx, int64_t j0, F val) {
  const int4 ia = __ldg(reinterpret_cast<const int4*>(idx + j0));
  const int4 ib = __ldg(reinterpret_cast<const int4*>(idx + j0 + 4));
  __nv_bfloat162 p0 = __floats2bfloat162_rn(val(ia.x, j0 + 0), val(ia.y, j0 + 1));
  __nv_bfloat162 p1 = __floats2bfloat162_rn(val(ia.z, j0 + 2), val(ia.w, j0 + 3));
  __nv_bfloat162 p2 = __floats2bfloat162_rn(val(ib.x, j0 + 4), val(ib.y, j0 + 5));
  __nv_bfloat162 p3 = __floats2bfloat162_rn(val(ib.z, j0 + 6), val(ib.w, j0 + 7));
  uint4 v;
  v.x = *reinterpret_cast<uint32_t*>(&p0);
  v.y = *reinterpret_cast<uint32_t*>(&p1);
  v.z = *reinterpret_cast<uint32_t*>(&p2);
  v.w = *reinterpret_cast<uint32_t*>(&p3);
  return v;
}

__global__ void __launch_bounds__(kThreads) rmsnorm_gather_kernel(
    int64_t T, int64_t d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    float eps, int K, IdxList outs, float* __restrict__ rstd_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);
  float* red = reinterpret_cast<float*>(sm + d * 2);
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(xs, x + r * d, d);
    __syncthreads();
    float ss = 0.f;
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
      float v = bf(xs[c]);
      ss += v * v;
    }
    const float rstd = rsqrtf(block_sum(ss, red) / static_cast<float>(d) + eps);
    if (threadIdx.x == 0) rstd_out[r] = rstd;
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x)
      xs[c] = __float2bfloat16_rn(bf(xs[c]) * rstd * w[c]);
    __syncthreads();
    for (int k = 0; k < K; ++k) {
      uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(outs.ptr[k]) + r * d);
      for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x)
        __stcs(dst + i, gather8(outs.idx[k], 8 * i, [&](int c, int64_t) { return bf(xs[c]); }));
    }
    __syncthreads();
  }
}

// dy[c] = sum_k du_k[inv_k[c]];  g = dy*w ; dx = rstd*g - rstd^3 x (g.x)/d ;
// dw partial[c] += dy*x*rstd  (per CTA, reduced later in fixed order)
__global__ void __launch_bounds__(kThreads) rmsnorm_gather_bwd_kernel(
    int64_t T, int64_t d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    const float* __restrict__ rstd_in, int K, IdxList dus, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dw_part) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* dus_s = xs + d;                       // K rows
  float* dy = reinterpret_cast<float*>(dus_s + K * d);  // fp32 row
  float* red = dy + d;
  float dwacc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) dwacc[i] = 0.f;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(xs, x + r * d, d);
    for (int k = 0; k < K; ++k)
      load_row(dus_s + k * d, static_cast<const __nv_bfloat16*>(dus.ptr[k]) + r * d, d);
    __syncthreads();
    const float rstd = rstd_in[r];
    float dot = 0.f;
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
      float s = 0.f;
      for (int k = 0; k < K; ++k) s += bf(dus_s[k * d + __ldg(dus.idx[k] + c)]);
      dy[c] = s;
      dot += s * w[c] * bf(xs[c]);
    }
    const float tot = block_sum(dot, red);
    const float coef = rstd * rstd * rstd * tot / static_cast<float>(d);
    int q = 0;
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x, ++q) {
      const float xv = bf(xs[c]);
      dx[r * d + c] = __float2bfloat16_rn(rstd * dy[c] * w[c] - coef * xv);
      if (q < 16) dwacc[q] += dy[c] * xv * rstd;
    }
    __syncthreads();
  }
  int q = 0;
  for (int64_t c = threadIdx.x; c < d && q < 16; c += blockDim.x, ++q)
    dw_part[blockIdx.x * d + c] = dwacc[q];
}

__global__ void colsum_kernel(int64_t rows, int64_t d, const float* __restrict__ part,
                              float* __restrict__ out, int accumulate) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < d;
       c += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t r = 0; r < rows; ++r) s += part[r * d + c];  // fixed order
    out[c] = accumulate ? out[c] + s : s;
  }
}

__device__ __forceinline__ float silu_f(float v) { return v / (1.f + __expf(-v)); }
__device__ __forceinline__ float dsilu_f(float v) {
  const float s = 1.f / (1.f + __expf(-v));
  return s * (1.f + v * (1.f - s));
}

__global__ void __launch_bounds__(kThreads) swiglu_gather_kernel(
    int64_t T, int64_t f, const __nv_bfloat16* __restrict__ vg, const __nv_bfloat16* __restrict__ vu,
    const int32_t* __restrict__ cg, const int32_t* __restrict__ cu, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* gs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* us = gs + f;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(gs, vg + r * f, f);
    load_row(us, vu + r * f, f);
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(out + r * f);
    for (int64_t i = threadIdx.x; i < f / 8; i += blockDim.x) {
      const int4 ua = __ldg(reinterpret_cast<const int4*>(cu + 8 * i));
      const int4 ub = __ldg(reinterpret_cast<const int4*>(cu + 8 * i + 4));
      const int uidx[8] = {ua.x, ua.y, ua.z, ua.w, ub.x, ub.y, ub.z, ub.w};
      __stcs(dst + i, gather8(cg, 8 * i, [&](int c, int64_t j) {
               return silu_f(bf(gs[c])) * bf(us[uidx[j - 8 * i]]);
             }));
    }
    __syncthreads();
  }
}

// dv_g[j] = du[A[j]] * silu'(v_g[j]) * v_u[B[j]] ; dv_u[j] = du[C[j]] * silu(v_g[D[j]])
__global__ void __launch_bounds__(kThreads) swiglu_gather_bwd_kernel(
    int64_t T, int64_t f, const __nv_bfloat16* __restrict__ vg, const __nv_bfloat16* __restrict__ vu,
    const __nv_bfloat16* __restrict__ du, const int32_t* __restrict__ A,
    const int32_t* __restrict__ B, const int32_t* __restrict__ Cc, const int32_t* __restrict__ D,
    __nv_bfloat16* __restrict__ dvg, __nv_bfloat16* __restrict__ dvu) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* gs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* us = gs + f;
  __nv_bfloat16* ds = us + f;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(gs, vg + r * f, f);
    load_row(us, vu + r * f, f);
    load_row(ds, du + r * f, f);
    __syncthreads();
    uint4* og = reinterpret_cast<uint4*>(dvg + r * f);
    uint4* ou = reinterpret_cast<uint4*>(dvu + r * f);
    for (int64_t i = threadIdx.x; i < f / 8; i += blockDim.x) {
      const int4 ba = __ldg(reinterpret_cast<const int4*>(B + 8 * i));
      const int4 bb = __ldg(reinterpret_cast<const int4*>(B + 8 * i + 4));
      const int bidx[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
      __stcs(og + i, gather8(A, 8 * i, [&](int a, int64_t j) {
               return bf(ds[a]) * dsilu_f(bf(gs[j])) * bf(us[bidx[j - 8 * i]]);
             }));
      const int4 da = __ldg(reinterpret_cast<const int4*>(D + 8 * i));
      const int4 db = __ldg(reinterpret_cast<const int4*>(D + 8 * i + 4));
      const int didx[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
      __stcs(ou + i, gather8(Cc, 8 * i, [&](int c, int64_t j) {
               return bf(ds[c]) * silu_f(bf(gs[didx[j - 8 * i]]));
             }));
    }
    __syncthreads();
  }
}

// out = RoPE(z), z[c] = v[inv[c]]; pairs (c, c + hd/2) inside each head
__global__ void __launch_bounds__(kThreads) rope_scatter_kernel(
    int64_t T, int64_t S, int64_t H, int64_t hd, const __nv_bfloat16* __restrict__ v,
    const int32_t* __restrict__ inv, const float* __restrict__ cosb, const float* __restrict__ sinb,
    __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(sm);
  const int64_t d = H * hd, half = hd / 2;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(vs, v + r * d, d);
    __syncthreads();
    const int64_t s = r % S;
    for (int64_t p = threadIdx.x; p < d / 2; p += blockDim.x) {
      const int64_t h = p / half, i = p % half;
      const int64_t c1 = h * hd + i, c2 = c1 + half;
      const float z1 = bf(vs[__ldg(inv + c1)]), z2 = bf(vs[__ldg(inv + c2)]);
      const float cs = cosb[s * half + i], sn = sinb[s * half + i];
      out[r * d + c1] = __float2bfloat16_rn(z1 * cs - z2 * sn);
      out[r * d + c2] = __float2bfloat16_rn(z2 * cs + z1 * sn);
    }
    __syncthreads();
  }
}

// dz = RoPE^T(dout) ; dv[j] = dz[fwd[j]]
__global__ void __launch_bounds__(kThreads) rope_scatter_bwd_kernel(
    int64_t T, int64_t S, int64_t H, int64_t hd, const __nv_bfloat16* __restrict__ dout,
    const int32_t* __restrict__ fwd, const float* __restrict__ cosb, const float* __restrict__ sinb,
    __nv_bfloat16* __restrict__ dv) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* os = reinterpret_cast<__nv_bfloat16*>(sm);
  float* dz = reinterpret_cast<float*>(sm + H * hd * 2);
  const int64_t d = H * hd, half = hd / 2;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(os, dout + r * d, d);
    __syncthreads();
    const int64_t s = r % S;
    for (int64_t p = threadIdx.x; p < d / 2; p += blockDim.x) {
      const int64_t h = p / half, i = p % half;
      const int64_t c1 = h * hd + i, c2 = c1 + half;
      const float g1 = bf(os[c1]), g2 = bf(os[c2]);
      const float cs = cosb[s * half + i], sn = sinb[s * half + i];
      dz[c1] = g1 * cs + g2 * sn;
      dz[c2] = g2 * cs - g1 * sn;
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(dv + r * d);
    for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x)
      __stcs(dst + i, gather8(fwd, 8 * i, [&](int c, int64_t) { return dz[c]; }));
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) scatter_add_kernel(
    int64_t T, int64_t d, const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ v,
    const int32_t* __restrict__ inv, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(sm);
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    load_row(vs, v + r * d, d);
    __syncthreads();
    const uint4* hr = reinterpret_cast<const uint4*>(h + r * d);
    uint4* dst = reinterpret_cast<uint4*>(out + r * d);
    for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x) {
      uint4 hv = __ldcs(hr + i);
      const __nv_bfloat16* hh = reinterpret_cast<const __nv_bfloat16*>(&hv);
      __stcs(dst + i, gather8(inv, 8 * i, [&](int c, int64_t j) { return bf(hh[j - 8 * i]) + bf(vs[c]); }));
    }
    __syncthreads();
  }
}

int check_rows(int64_t T, int64_t d, size_t smem) {
  POETX_REQUIRE(T >= 0 && d > 0 && d % 8 == 0, POETX_ESHAPE, "row kernel: bad shape (%lld, %lld)",
                (long long)T, (long long)d);
  POETX_REQUIRE(smem <= 200 * 1024, POETX_ESHAPE, "row kernel: row too wide (%lld)", (long long)d);
  return POETX_OK;
}

unsigned row_grid(int64_t T) { return static_cast<unsigned>(T < 148 * 8 ? (T > 0 ? T : 1) : 148 * 8); }

template <typename K>
void set_smem(K kernel, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace
}  // namespace poetx

using namespace poetx;

extern "C" {

int poetx_rmsnorm_gather(int64_t T, int64_t d, const void* x, const float* w, float eps, int K,
                         const int32_t* const* idx, void* const* out, float* rstd, void* stream) {
  POETX_REQUIRE(K >= 1 && K <= kMaxK, POETX_ESHAPE, "rmsnorm_gather: 1..3 outputs");
  const size_t smem = d * 2 + 64 * 4;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  IdxList L{};
  for (int k = 0; k < K; ++k) { L.idx[k] = idx[k]; L.ptr[k] = out[k]; }
  set_smem(rmsnorm_gather_kernel, smem);
  rmsnorm_gather_kernel<<<row_grid(T), kThreads, smem, as_stream(stream)>>>(
      T, d, static_cast<const __nv_bfloat16*>(x), w, eps, K, L, rstd);
  POETX_LAUNCHED("rmsnorm_gather");
  return POETX_OK;
}

size_t poetx_rmsnorm_gather_bwd_workspace_bytes(int64_t T, int64_t d) {
  return static_cast<size_t>(row_grid(T)) * d * 4 + 256;
}

int poetx_rmsnorm_gather_bwd(int64_t T, int64_t d, const void* x, const float* w, const float* rstd,
                             int K, const int32_t* const* inv, const void* const* du, void* dx,
                             float* dw, int accumulate_dw, void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(K >= 1 && K <= kMaxK, POETX_ESHAPE, "rmsnorm_gather_bwd: 1..3 inputs");
  POETX_REQUIRE(d <= 16 * kThreads, POETX_ESHAPE, "rmsnorm_gather_bwd: d > %d", 16 * kThreads);
  const size_t smem = d * 2 * (1 + K) + d * 4 + 64 * 4;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  const unsigned grid = row_grid(T);
  POETX_REQUIRE(ws_bytes >= static_cast<size_t>(grid) * d * 4, POETX_ESHAPE,
                "rmsnorm_gather_bwd: workspace too small");
  IdxList L{};
  for (int k = 0; k < K; ++k) { L.idx[k] = inv[k]; L.ptr[k] = const_cast<void*>(du[k]); }
  cudaStream_t st = as_stream(stream);
  set_smem(rmsnorm_gather_bwd_kernel, smem);
  float* part = static_cast<float*>(ws);
  rmsnorm_gather_bwd_kernel<<<grid, kThreads, smem, st>>>(
      T, d, static_cast<const __nv_bfloat16*>(x), w, rstd, K, L, static_cast<__nv_bfloat16*>(dx), part);
  POETX_LAUNCHED("rmsnorm_gather_bwd");
  colsum_kernel<<<grid_for(d, 256), 256, 0, st>>>(grid, d, part, dw, accumulate_dw);
  POETX_LAUNCHED("colsum");
  return POETX_OK;
}

int poetx_swiglu_gather(int64_t T, int64_t f, const void* vg, const void* vu, const int32_t* cg,
                        const int32_t* cu, void* out, void* stream) {
  const size_t smem = 2 * f * 2;
  POETX_TRY(check_rows(T, f, smem));
  if (T == 0) return POETX_OK;
  set_smem(swiglu_gather_kernel, smem);
  swiglu_gather_kernel<<<row_grid(T), kThreads, smem, as_stream(stream)>>>(
      T, f, static_cast<const __nv_bfloat16*>(vg), static_cast<const __nv_bfloat16*>(vu), cg, cu,
      static_cast<__nv_bfloat16*>(out));
  POETX_LAUNCHED("swiglu_gather");
  return POETX_OK;
}

int poetx_swiglu_gather_bwd(int64_t T, int64_t f, const void* vg, const void* vu, const void* du,
                            const int32_t* A, const int32_t* B, const int32_t* Cc, const int32_t* D,
                            void* dvg, void* dvu, void* stream) {
  const size_t smem = 3 * f * 2;
  POETX_TRY(check_rows(T, f, smem));
  if (T == 0) return POETX_OK;
  set_smem(swiglu_gather_bwd_kernel, smem);
  swiglu_gather_bwd_kernel<<<row_grid(T), kThreads, smem, as_stream(stream)>>>(
      T, f, static_cast<const __nv_bfloat16*>(vg), static_cast<const __nv_bfloat16*>(vu),
      static_cast<const __nv_bfloat16*>(du), A, B, Cc, D, static_cast<__nv_bfloat16*>(dvg),
      static_cast<__nv_bfloat16*>(dvu));
  POETX_LAUNCHED("swiglu_gather_bwd");
  return POETX_OK;
}

int poetx_rope_scatter(int64_t T, int64_t S, int64_t H, int64_t hd, const void* v,
                       const int32_t* inv, const float* cosb, const float* sinb, void* out,
                       void* stream) {
  POETX_REQUIRE(hd % 2 == 0 && S > 0, POETX_ESHAPE, "rope_scatter: bad head dim / seq");
  const size_t smem = H * hd * 2;
  POETX_TRY(check_rows(T, H * hd, smem));
  if (T == 0) return POETX_OK;
  set_smem(rope_scatter_kernel, smem);
  rope_scatter_kernel<<<row_grid(T), kThreads, smem, as_stream(stream)>>>(
      T, S, H, hd, static_cast<const __nv_bfloat16*>(v), inv, cosb, sinb,
      static_cast<__nv_bfloat16*>(out));
  POETX_LAUNCHED("rope_scatter");
  return POETX_OK;
}

int poetx_rope_scatter_bwd(int64_t T, int64_t S, int64_t H, int64_t hd, const void* dout,
                           const int32_t* fwd, const float* cosb, const float* sinb, void* dv,
                           void* stream) {
  POETX_REQUIRE(hd % 2 == 0 && S > 0, POETX_ESHAPE, "rope_scatter_bwd: bad head dim / seq");
  const size_t smem = H * hd * 2 + H * hd * 4;
  POETX_TRY(check_rows(T, H * hd, smem));
  if (T == 0) return POETX_OK;
  set_smem(rope_scatter_bwd_kernel, smem);
  rope_scatter_bwd_kernel<<<row_grid(T), kThreads, smem, as_stream(stream)>>>(
      T, S, H, hd, static_cast<const __nv_bfloat16*>(dout), fwd, cosb, sinb,
      static_cast<__nv_bfloat16*>(dv));
  POETX_LAUNCHED("rope_scatter_bwd");
  return POETX_OK;
}

int poetx_scatter_add(int64_t T, int64_t d, const void* h, const void* v, const int32_t* inv,
                      void* out, void* stream) {
  const size_t smem = d * 2;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  set_smem(scatter_add_kernel, smem);
  scatter_add_kernel<<<row_grid(T), kThreads, smem, as_stream(stream)>>>(
      T, d, static_cast<const __nv_bfloat16*>(h), static_cast<const __nv_bfloat16*>(v), inv,
      static_cast<__nv_bfloat16*>(out));
  POETX_LAUNCHED("scatter_add");
  return POETX_OK;
}

}  // extern "C"
