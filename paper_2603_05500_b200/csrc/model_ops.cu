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
// Tiles of rows per CTA iteration (grid-stride), staged in shared memory with
// 16-byte coalesced loads, outputs written with 16-byte coalesced stores.
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// All kernels process TILES of RT rows per iteration: the rows are staged in
// shared memory with 16-byte loads, and every index vector (8 columns per
// int4 pair) is loaded once per tile and applied to all RT rows.
// ---------------------------------------------------------------------------

template <int RT>
__device__ __forceinline__ int64_t tile_rows(int64_t r0, int64_t T) { return T - r0 < RT ? T - r0 : RT; }

__device__ __forceinline__ void load_rows(__nv_bfloat16* s, const __nv_bfloat16* g, int64_t nrows,
                                          int64_t n) {
  const uint4* src = reinterpret_cast<const uint4*>(g);
  uint4* dst = reinterpret_cast<uint4*>(s);
  for (int64_t i = threadIdx.x; i < nrows * (n / 8); i += blockDim.x) dst[i] = __ldcs(src + i);
}

__device__ __forceinline__ void load_idx8(const int32_t* idx, int64_t j0, int (&o)[8]) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(idx + j0));
  const int4 b = __ldg(reinterpret_cast<const int4*>(idx + j0 + 4));
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]);
  __nv_bfloat162 p1 = __floats2bfloat162_rn(v[2], v[3]);
  __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]);
  __nv_bfloat162 p3 = __floats2bfloat162_rn(v[6], v[7]);
  uint4 u;
  u.x = *reinterpret_cast<uint32_t*>(&p0);
  u.y = *reinterpret_cast<uint32_t*>(&p1);
  u.z = *reinterpret_cast<uint32_t*>(&p2);
  u.w = *reinterpret_cast<uint32_t*>(&p3);
  return u;
}

// per-row sum of squares: warp w reduces rows w, w + 8, ...
__device__ __forceinline__ void rows_rstd(const __nv_bfloat16* xs, int64_t nrows, int64_t d, float eps,
                                          float* rstd_s) {
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int64_t r = w; r < nrows; r += blockDim.x / 32) {
    float ss = 0.f;
    for (int64_t c = l; c < d; c += 32) {
      const float v = bf(xs[r * d + c]);
      ss += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (l == 0) rstd_s[r] = rsqrtf(ss / static_cast<float>(d) + eps);
  }
}

template <int RT>
__global__ void __launch_bounds__(kThreads) rmsnorm_gather_kernel(
    int64_t T, int64_t d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    float eps, int K, IdxList outs, float* __restrict__ rstd_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);
  float* rstd_s = reinterpret_cast<float*>(sm + RT * d * 2);
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(xs, x + r0 * d, nr, d);
    __syncthreads();
    rows_rstd(xs, nr, d, eps, rstd_s);
    __syncthreads();
    for (int64_t e = threadIdx.x; e < nr * d; e += blockDim.x) {
      const int64_t r = e / d, c = e % d;
      xs[e] = __float2bfloat16_rn(bf(xs[e]) * rstd_s[r] * w[c]);
    }
    if (threadIdx.x < nr) rstd_out[r0 + threadIdx.x] = rstd_s[threadIdx.x];
    __syncthreads();
    for (int k = 0; k < K; ++k) {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(outs.ptr[k]) + r0 * d;
      for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x) {
        int id[8];
        load_idx8(outs.idx[k], 8 * i, id);
        for (int64_t r = 0; r < nr; ++r) {
          float v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = bf(xs[r * d + id[q]]);
          __stcs(reinterpret_cast<uint4*>(o + r * d) + i, pack8(v));
        }
      }
    }
    __syncthreads();
  }
}

// dy = sum_k du_k[:, inv_k]; g = dy*w ; dx = rstd*g - rstd^3 x (g.x)/d ;
// dw partial[c] += dy*x*rstd  (per CTA, reduced later in fixed order)
template <int RT>
__global__ void __launch_bounds__(kThreads) rmsnorm_gather_bwd_kernel(
    int64_t T, int64_t d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    const float* __restrict__ rstd_in, int K, IdxList dus, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dw_part) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);   // RT rows
  __nv_bfloat16* dus_s = xs + RT * d;                         // K x RT rows
  float* dy = reinterpret_cast<float*>(dus_s + K * RT * d);    // RT rows fp32
  float* dot_s = dy + RT * d;                                  // RT
  float dwacc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) dwacc[i] = 0.f;
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(xs, x + r0 * d, nr, d);
    for (int k = 0; k < K; ++k)
      load_rows(dus_s + k * RT * d, static_cast<const __nv_bfloat16*>(dus.ptr[k]) + r0 * d, nr, d);
    __syncthreads();
    // dy (gathers amortised over the tile's rows)
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
      int iv[kMaxK];
      for (int k = 0; k < K; ++k) iv[k] = __ldg(dus.idx[k] + c);
      for (int64_t r = 0; r < nr; ++r) {
        float s = 0.f;
        for (int k = 0; k < K; ++k) s += bf(dus_s[(k * RT + r) * d + iv[k]]);
        dy[r * d + c] = s;
      }
    }
    __syncthreads();
    for (int64_t r = wp; r < nr; r += blockDim.x / 32) {
      float acc = 0.f;
      for (int64_t c = l; c < d; c += 32) acc += dy[r * d + c] * w[c] * bf(xs[r * d + c]);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (l == 0) dot_s[r] = acc;
    }
    __syncthreads();
    int q = 0;
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x, ++q) {
      const float wc = w[c];
      float dwc = 0.f;
      for (int64_t r = 0; r < nr; ++r) {
        const float rs = rstd_in[r0 + r];
        const float xv = bf(xs[r * d + c]);
        const float coef = rs * rs * rs * dot_s[r] / static_cast<float>(d);
        dx[(r0 + r) * d + c] = __float2bfloat16_rn(rs * dy[r * d + c] * wc - coef * xv);
        dwc += dy[r * d + c] * xv * rs;
      }
      if (q < 16) dwacc[q] += dwc;
    }
    __syncthreads();
  }
  int q = 0;
  for (int64_t c = threadIdx.x; c < d && q < 16; c += blockDim.x, ++q)
    dw_part[blockIdx.x * d + c] = dwacc[q];
}

// column sums of a [rows, d] partial matrix: 8 warps split the rows of a
// 32-column strip, fixed-order combine in smem (deterministic)
__global__ void __launch_bounds__(256) colsum_kernel(int64_t rows, int64_t d, const float* __restrict__ part,
                                                     float* __restrict__ out, int accumulate) {
  __shared__ float red[8][33];
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32; c0 < d; c0 += static_cast<int64_t>(gridDim.x) * 32) {
    const int64_t c = c0 + l;
    float s = 0.f;
    if (c < d)
      for (int64_t r = wp; r < rows; r += 8) s += part[r * d + c];
    red[wp][l] = s;
    __syncthreads();
    if (wp == 0 && c < d) {
      float t = 0.f;
      for (int k = 0; k < 8; ++k) t += red[k][l];
      out[c] = accumulate ? out[c] + t : t;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ float silu_f(float v) { return v / (1.f + __expf(-v)); }
__device__ __forceinline__ float dsilu_f(float v) {
  const float s = 1.f / (1.f + __expf(-v));
  return s * (1.f + v * (1.f - s));
}

template <int RT>
__global__ void __launch_bounds__(kThreads) swiglu_gather_kernel(
    int64_t T, int64_t f, const __nv_bfloat16* __restrict__ vg, const __nv_bfloat16* __restrict__ vu,
    const int32_t* __restrict__ cg, const int32_t* __restrict__ cu, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* gs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* us = gs + RT * f;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(gs, vg + r0 * f, nr, f);
    load_rows(us, vu + r0 * f, nr, f);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < f / 8; i += blockDim.x) {
      int ig[8], iu[8];
      load_idx8(cg, 8 * i, ig);
      load_idx8(cu, 8 * i, iu);
      for (int64_t r = 0; r < nr; ++r) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = silu_f(bf(gs[r * f + ig[q]])) * bf(us[r * f + iu[q]]);
        __stcs(reinterpret_cast<uint4*>(out + (r0 + r) * f) + i, pack8(v));
      }
    }
    __syncthreads();
  }
}

// dv_g[j] = du[A[j]] * silu'(v_g[j]) * v_u[B[j]] ; dv_u[j] = du[C[j]] * silu(v_g[D[j]])
template <int RT>
__global__ void __launch_bounds__(kThreads) swiglu_gather_bwd_kernel(
    int64_t T, int64_t f, const __nv_bfloat16* __restrict__ vg, const __nv_bfloat16* __restrict__ vu,
    const __nv_bfloat16* __restrict__ du, const int32_t* __restrict__ A,
    const int32_t* __restrict__ B, const int32_t* __restrict__ Cc, const int32_t* __restrict__ D,
    __nv_bfloat16* __restrict__ dvg, __nv_bfloat16* __restrict__ dvu) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* gs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* us = gs + RT * f;
  __nv_bfloat16* ds = us + RT * f;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(gs, vg + r0 * f, nr, f);
    load_rows(us, vu + r0 * f, nr, f);
    load_rows(ds, du + r0 * f, nr, f);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < f / 8; i += blockDim.x) {
      int ia[8], ib[8], ic[8], id[8];
      load_idx8(A, 8 * i, ia);
      load_idx8(B, 8 * i, ib);
      load_idx8(Cc, 8 * i, ic);
      load_idx8(D, 8 * i, id);
      for (int64_t r = 0; r < nr; ++r) {
        const int64_t o = r * f;
        float g[8], u[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          g[q] = bf(ds[o + ia[q]]) * dsilu_f(bf(gs[o + 8 * i + q])) * bf(us[o + ib[q]]);
          u[q] = bf(ds[o + ic[q]]) * silu_f(bf(gs[o + id[q]]));
        }
        __stcs(reinterpret_cast<uint4*>(dvg + (r0 + r) * f) + i, pack8(g));
        __stcs(reinterpret_cast<uint4*>(dvu + (r0 + r) * f) + i, pack8(u));
      }
    }
    __syncthreads();
  }
}

// out = RoPE(z), z[c] = v[inv[c]]; 8 outputs per vector all lie in one half of a head
template <int RT>
__global__ void __launch_bounds__(kThreads) rope_scatter_kernel(
    int64_t T, int64_t S, int64_t H, int64_t hd, const __nv_bfloat16* __restrict__ v,
    const int32_t* __restrict__ inv, const float* __restrict__ cosb, const float* __restrict__ sinb,
    __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(sm);
  const int64_t d = H * hd, half = hd / 2;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(vs, v + r0 * d, nr, d);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x) {
      const int64_t c0 = 8 * i, hh = c0 / hd, wi = c0 % hd;
      const bool first = wi < half;
      const int64_t pc0 = first ? c0 + half : c0 - half;  // partner columns
      const int64_t i0 = first ? wi : wi - half;          // frequency index
      int me[8], pa[8];
      load_idx8(inv, c0, me);
      load_idx8(inv, pc0, pa);
      (void)hh;
      for (int64_t r = 0; r < nr; ++r) {
        const int64_t s = (r0 + r) % S;
        float o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float cs = cosb[s * half + i0 + q], sn = sinb[s * half + i0 + q];
          const float zm = bf(vs[r * d + me[q]]), zp = bf(vs[r * d + pa[q]]);
          o[q] = first ? zm * cs - zp * sn : zm * cs + zp * sn;
        }
        __stcs(reinterpret_cast<uint4*>(out + (r0 + r) * d) + i, pack8(o));
      }
    }
    __syncthreads();
  }
}

// dv[j] = dz[fwd[j]], dz = RoPE^T(dout) computed on the fly from the staged row
template <int RT>
__global__ void __launch_bounds__(kThreads) rope_scatter_bwd_kernel(
    int64_t T, int64_t S, int64_t H, int64_t hd, const __nv_bfloat16* __restrict__ dout,
    const int32_t* __restrict__ fwd, const float* __restrict__ cosb, const float* __restrict__ sinb,
    __nv_bfloat16* __restrict__ dv) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* os = reinterpret_cast<__nv_bfloat16*>(sm);
  const int64_t d = H * hd, half = hd / 2;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(os, dout + r0 * d, nr, d);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x) {
      int cc[8];
      load_idx8(fwd, 8 * i, cc);
      for (int64_t r = 0; r < nr; ++r) {
        const int64_t s = (r0 + r) % S;
        float o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t c = cc[q], wi = c % hd;
          const bool first = wi < half;
          const int64_t fi = first ? wi : wi - half;
          const float cs = cosb[s * half + fi], sn = sinb[s * half + fi];
          const float g = bf(os[r * d + c]), gp = bf(os[r * d + (first ? c + half : c - half)]);
          o[q] = first ? g * cs + gp * sn : g * cs - gp * sn;
        }
        __stcs(reinterpret_cast<uint4*>(dv + (r0 + r) * d) + i, pack8(o));
      }
    }
    __syncthreads();
  }
}

template <int RT>
__global__ void __launch_bounds__(kThreads) scatter_add_kernel(
    int64_t T, int64_t d, const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ v,
    const int32_t* __restrict__ inv, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(sm);
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int64_t nr = tile_rows<RT>(r0, T);
    load_rows(vs, v + r0 * d, nr, d);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < d / 8; i += blockDim.x) {
      int id[8];
      load_idx8(inv, 8 * i, id);
      for (int64_t r = 0; r < nr; ++r) {
        uint4 hv = __ldcs(reinterpret_cast<const uint4*>(h + (r0 + r) * d) + i);
        const __nv_bfloat16* hh = reinterpret_cast<const __nv_bfloat16*>(&hv);
        float o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = bf(hh[q]) + bf(vs[r * d + id[q]]);
        __stcs(reinterpret_cast<uint4*>(out + (r0 + r) * d) + i, pack8(o));
      }
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

// rows per tile: ~48 KB of staged rows per CTA (index loads amortised over
// the tile, several CTAs per SM for latency hiding)
int pick_rt(int64_t bytes_per_row) {
  static int64_t budget = [] {
    const char* e = getenv("POETX_ROW_TILE_KB");
    return static_cast<int64_t>(e ? atoi(e) : 48) * 1024;
  }();
  int64_t rt = budget / (bytes_per_row > 0 ? bytes_per_row : 1);
  if (rt >= 8) return 8;
  if (rt >= 4) return 4;
  if (rt >= 2) return 2;
  return 1;
}
unsigned row_grid(int64_t T, int rt) {
  int64_t tiles = (T + rt - 1) / rt;
  return static_cast<unsigned>(tiles < 148 * 4 ? (tiles > 0 ? tiles : 1) : 148 * 4);
}
#define POETX_RT_DISPATCH(rt, KERNEL, ...)                    \
  switch (rt) {                                               \
    case 8: { auto k = KERNEL<8>; __VA_ARGS__; break; }       \
    case 4: { auto k = KERNEL<4>; __VA_ARGS__; break; }       \
    case 2: { auto k = KERNEL<2>; __VA_ARGS__; break; }       \
    default: { auto k = KERNEL<1>; __VA_ARGS__; break; }      \
  }

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
  const int rt = pick_rt(d * 2);
  const size_t smem = rt * d * 2 + 64 * 4;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  IdxList L{};
  for (int k = 0; k < K; ++k) { L.idx[k] = idx[k]; L.ptr[k] = out[k]; }
  POETX_RT_DISPATCH(rt, rmsnorm_gather_kernel, set_smem(k, smem);
                    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                        T, d, static_cast<const __nv_bfloat16*>(x), w, eps, K, L, rstd));
  POETX_LAUNCHED("rmsnorm_gather");
  return POETX_OK;
}

static int bwd_rt(int64_t d, int K) { return pick_rt(d * 2 * (1 + K) + d * 4); }

size_t poetx_rmsnorm_gather_bwd_workspace_bytes(int64_t T, int64_t d) {
  int rt = bwd_rt(d, 1);  // largest grid over K
  return static_cast<size_t>(row_grid(T, rt)) * d * 4 + 256;
}

int poetx_rmsnorm_gather_bwd(int64_t T, int64_t d, const void* x, const float* w, const float* rstd,
                             int K, const int32_t* const* inv, const void* const* du, void* dx,
                             float* dw, int accumulate_dw, void* ws, size_t ws_bytes, void* stream) {
  POETX_REQUIRE(K >= 1 && K <= kMaxK, POETX_ESHAPE, "rmsnorm_gather_bwd: 1..3 inputs");
  POETX_REQUIRE(d <= 16 * kThreads, POETX_ESHAPE, "rmsnorm_gather_bwd: d > %d", 16 * kThreads);
  const int rt = bwd_rt(d, K);
  const size_t smem = rt * d * 2 * (1 + K) + rt * d * 4 + 64 * 4;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  const unsigned grid = row_grid(T, rt);
  POETX_REQUIRE(ws_bytes >= static_cast<size_t>(grid) * d * 4, POETX_ESHAPE,
                "rmsnorm_gather_bwd: workspace too small");
  IdxList L{};
  for (int k = 0; k < K; ++k) { L.idx[k] = inv[k]; L.ptr[k] = const_cast<void*>(du[k]); }
  cudaStream_t st = as_stream(stream);
  float* part = static_cast<float*>(ws);
  POETX_RT_DISPATCH(rt, rmsnorm_gather_bwd_kernel, set_smem(k, smem);
                    k<<<grid, kThreads, smem, st>>>(T, d, static_cast<const __nv_bfloat16*>(x), w, rstd,
                                                    K, L, static_cast<__nv_bfloat16*>(dx), part));
  POETX_LAUNCHED("rmsnorm_gather_bwd");
  colsum_kernel<<<static_cast<unsigned>((d + 31) / 32), 256, 0, st>>>(grid, d, part, dw, accumulate_dw);
  POETX_LAUNCHED("colsum");
  return POETX_OK;
}

int poetx_swiglu_gather(int64_t T, int64_t f, const void* vg, const void* vu, const int32_t* cg,
                        const int32_t* cu, void* out, void* stream) {
  const int rt = pick_rt(2 * f * 2);
  const size_t smem = rt * 2 * f * 2;
  POETX_TRY(check_rows(T, f, smem));
  if (T == 0) return POETX_OK;
  POETX_RT_DISPATCH(rt, swiglu_gather_kernel, set_smem(k, smem);
                    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                        T, f, static_cast<const __nv_bfloat16*>(vg), static_cast<const __nv_bfloat16*>(vu),
                        cg, cu, static_cast<__nv_bfloat16*>(out)));
  POETX_LAUNCHED("swiglu_gather");
  return POETX_OK;
}

int poetx_swiglu_gather_bwd(int64_t T, int64_t f, const void* vg, const void* vu, const void* du,
                            const int32_t* A, const int32_t* B, const int32_t* Cc, const int32_t* D,
                            void* dvg, void* dvu, void* stream) {
  const int rt = pick_rt(3 * f * 2);
  const size_t smem = rt * 3 * f * 2;
  POETX_TRY(check_rows(T, f, smem));
  if (T == 0) return POETX_OK;
  POETX_RT_DISPATCH(rt, swiglu_gather_bwd_kernel, set_smem(k, smem);
                    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                        T, f, static_cast<const __nv_bfloat16*>(vg), static_cast<const __nv_bfloat16*>(vu),
                        static_cast<const __nv_bfloat16*>(du), A, B, Cc, D,
                        static_cast<__nv_bfloat16*>(dvg), static_cast<__nv_bfloat16*>(dvu)));
  POETX_LAUNCHED("swiglu_gather_bwd");
  return POETX_OK;
}

int poetx_rope_scatter(int64_t T, int64_t S, int64_t H, int64_t hd, const void* v,
                       const int32_t* inv, const float* cosb, const float* sinb, void* out,
                       void* stream) {
  POETX_REQUIRE(hd % 2 == 0 && S > 0 && (hd / 2) % 8 == 0, POETX_ESHAPE,
                "rope_scatter: head_dim/2 must be a multiple of 8, seq > 0");
  const int rt = pick_rt(H * hd * 2);
  const size_t smem = rt * H * hd * 2;
  POETX_TRY(check_rows(T, H * hd, smem));
  if (T == 0) return POETX_OK;
  POETX_RT_DISPATCH(rt, rope_scatter_kernel, set_smem(k, smem);
                    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                        T, S, H, hd, static_cast<const __nv_bfloat16*>(v), inv, cosb, sinb,
                        static_cast<__nv_bfloat16*>(out)));
  POETX_LAUNCHED("rope_scatter");
  return POETX_OK;
}

int poetx_rope_scatter_bwd(int64_t T, int64_t S, int64_t H, int64_t hd, const void* dout,
                           const int32_t* fwd, const float* cosb, const float* sinb, void* dv,
                           void* stream) {
  POETX_REQUIRE(hd % 2 == 0 && S > 0, POETX_ESHAPE, "rope_scatter_bwd: bad head dim / seq");
  const int rt = pick_rt(H * hd * 2);
  const size_t smem = rt * H * hd * 2;
  POETX_TRY(check_rows(T, H * hd, smem));
  if (T == 0) return POETX_OK;
  POETX_RT_DISPATCH(rt, rope_scatter_bwd_kernel, set_smem(k, smem);
                    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                        T, S, H, hd, static_cast<const __nv_bfloat16*>(dout), fwd, cosb, sinb,
                        static_cast<__nv_bfloat16*>(dv)));
  POETX_LAUNCHED("rope_scatter_bwd");
  return POETX_OK;
}

int poetx_scatter_add(int64_t T, int64_t d, const void* h, const void* v, const int32_t* inv,
                      void* out, void* stream) {
  const int rt = pick_rt(d * 2);
  const size_t smem = rt * d * 2;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  POETX_RT_DISPATCH(rt, scatter_add_kernel, set_smem(k, smem);
                    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                        T, d, static_cast<const __nv_bfloat16*>(h), static_cast<const __nv_bfloat16*>(v),
                        inv, static_cast<__nv_bfloat16*>(out)));
  POETX_LAUNCHED("scatter_add");
  return POETX_OK;
}

}  // extern "C"
