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
#include "tile8.cuh"

#ifndef POETX_ROW_PROBE
#define POETX_ROW_PROBE 0
#endif
namespace poetx {
namespace {

constexpr int kThreads = 256;
constexpr int kColsumSplits = 16;  // stage-1 row splits of the RMSNorm dw column sum
constexpr int kMaxK = 3;

struct IdxList {
  const int32_t* idx[kMaxK];
  void* ptr[kMaxK];
};

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// ---------------------------------------------------------------------------
// All kernels process TILES of RT rows per iteration: the rows are staged in
// shared memory with cp.async 16-byte copies, every index vector (8 columns
// per int4 pair) is loaded once per tile and applied to all RT rows, and all
// global stores are 16-byte vectors.  In-row offsets are 32-bit.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// stage nrows consecutive rows of n bf16 (n % 8 == 0) into smem
__device__ __forceinline__ void stage_rows(__nv_bfloat16* s, const __nv_bfloat16* g, int nrows, int n) {
  const uint4* src = reinterpret_cast<const uint4*>(g);
  uint4* dst = reinterpret_cast<uint4*>(s);
  const int nv = nrows * (n / 8);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) cp16(dst + i, src + i);
}

__device__ __forceinline__ void load_idx8(const int32_t* idx, int j0, int (&o)[8]) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(idx + j0));
  const int4 b = __ldg(reinterpret_cast<const int4*>(idx + j0 + 4));
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
// 16-bit index maps (features < 65536): half the index bytes through L1,
// which is what the SwiGLU kernels' L1/shared pipe saturates on
__device__ __forceinline__ void load_idx8(const uint16_t* idx, int j0, int (&o)[8]) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(idx + j0));
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    o[2 * q] = static_cast<int>(w[q] & 0xFFFFu);
    o[2 * q + 1] = static_cast<int>(w[q] >> 16);
  }
}
__device__ __forceinline__ void load_f8(const float* p, float (&o)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void unpack8(const uint4 u, float (&o)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __bfloat1622float2(h[q]);
    o[2 * q] = f.x;
    o[2 * q + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat162 p = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    w[q] = *reinterpret_cast<uint32_t*>(&p);
  }
  return u;
}
__device__ __forceinline__ float sigmoid_f(float v) { return __frcp_rn(1.f + __expf(-v)); }

// K (number of consumers) is a template parameter: the IdxList entries and
// per-consumer index registers must be compile-time indexed (else local memory)
template <int RT, int K>
__global__ void __launch_bounds__(kThreads) rmsnorm_gather_kernel(
    int64_t T, int d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    float eps, IdxList outs, float* __restrict__ rstd_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);
  float* rstd_s = reinterpret_cast<float*>(sm + RT * d * 2);
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32, nvec = d / 8;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(xs, x + r0 * d, nr, d);
    cp_wait_all();
    __syncthreads();
    for (int r = wp; r < nr; r += kThreads / 32) {  // warp per row: sum of squares
      float ss = 0.f;
      const uint4* row = reinterpret_cast<const uint4*>(xs + r * d);
      for (int i = l; i < nvec; i += 32) {
        float v[8];
        unpack8(row[i], v);
#pragma unroll
        for (int q = 0; q < 8; ++q) ss += v[q] * v[q];
      }
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (l == 0) rstd_s[r] = rsqrtf(ss / static_cast<float>(d) + eps);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nvec; i += kThreads) {  // y = x * rstd * w in place
      float wv[8];
      load_f8(w + 8 * i, wv);
      for (int r = 0; r < nr; ++r) {
        uint4* p = reinterpret_cast<uint4*>(xs + r * d) + i;
        float v[8];
        unpack8(*p, v);
        const float rs = rstd_s[r];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = v[q] * rs * wv[q];
        *p = pack8(v);
      }
    }
    if (threadIdx.x < nr) rstd_out[r0 + threadIdx.x] = rstd_s[threadIdx.x];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(outs.ptr[k]) + r0 * d;
      for (int i = threadIdx.x; i < nvec; i += kThreads) {
        int id[8];
        load_idx8(outs.idx[k], 8 * i, id);
        for (int r = 0; r < nr; ++r) {
          const __nv_bfloat16* row = xs + r * d;
          float v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = bf(row[id[q]]);
          __stcs(reinterpret_cast<uint4*>(o + static_cast<int64_t>(r) * d) + i, pack8(v));
        }
      }
    }
    __syncthreads();
  }
}

// dy = sum_k du_k[:, inv_k]; g = dy*w ; dx = rstd*g - rstd^3 x (g.x)/d ;
// dw partial[c] += dy*x*rstd  (per CTA, reduced later in fixed order)
template <int RT, int K>
__global__ void __launch_bounds__(kThreads) rmsnorm_gather_bwd_kernel(
    int64_t T, int d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    const float* __restrict__ rstd_in, IdxList dus, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ dw_part) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);   // RT rows
  __nv_bfloat16* dus_s = xs + RT * d;                         // K x RT rows
  float* dy = reinterpret_cast<float*>(dus_s + K * RT * d);    // RT rows fp32
  float* red = dy + RT * d;                                    // [RT][8] warp partials
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32, nvec = d / 8;
  float dwacc[2][8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 8; ++q) dwacc[a][q] = 0.f;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(xs, x + r0 * d, nr, d);
#pragma unroll
    for (int k = 0; k < K; ++k)
      stage_rows(dus_s + k * RT * d, static_cast<const __nv_bfloat16*>(dus.ptr[k]) + r0 * d, nr, d);
    // the second pass's global reads (residual gradient, rstd) issued now, so
    // their latency hides under the staging and the first pass instead of
    // stalling every row of the second pass
    uint4 resv[2][RT];
    float rsv[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      rsv[r] = r < nr ? rstd_in[r0 + r] : 0.f;
#pragma unroll
      for (int slot = 0; slot < 2; ++slot) {
        const int i = threadIdx.x + slot * kThreads;
        resv[slot][r] = (dres && r < nr && i < nvec)
                            ? __ldcs(reinterpret_cast<const uint4*>(dres + (r0 + r) * d) + i)
                            : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    cp_wait_all();
    __syncthreads();
    float dot[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) dot[r] = 0.f;
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      int iv[K][8];
#pragma unroll
      for (int k = 0; k < K; ++k) load_idx8(dus.idx[k], 8 * i, iv[k]);
#if POETX_ROW_PROBE == 1  // timing probe: conflict-free identity gathers (results invalid)
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < 8; ++q) iv[k][q] = (8 * i + q) ^ (iv[k][q] & 0);
#endif
      float wv[8];
      load_f8(w + 8 * i, wv);
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        if (r >= nr) break;
        float s[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const __nv_bfloat16* row = dus_s + (k * RT + r) * d;
#pragma unroll
          for (int q = 0; q < 8; ++q) s[q] += bf(row[iv[k][q]]);
        }
        float xv[8];
        unpack8(reinterpret_cast<const uint4*>(xs + r * d)[i], xv);
        float4* dyp = reinterpret_cast<float4*>(dy + r * d + 8 * i);
        dyp[0] = make_float4(s[0], s[1], s[2], s[3]);
        dyp[1] = make_float4(s[4], s[5], s[6], s[7]);
#pragma unroll
        for (int q = 0; q < 8; ++q) dot[r] += s[q] * wv[q] * xv[q];
      }
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      float v = dot[r];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0) red[r * 8 + wp] = v;
    }
    __syncthreads();
#pragma unroll
    for (int slot = 0; slot < 2; ++slot) {  // compile-time slot: dwacc stays in registers
      const int i = threadIdx.x + slot * kThreads;
      if (i >= nvec) break;
      float wv[8];
      load_f8(w + 8 * i, wv);
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        if (r >= nr) break;
        float tot = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) tot += red[r * 8 + k];
        const float rs = rsv[r];
        const float coef = rs * rs * rs * tot / static_cast<float>(d);
        float xv[8], o[8], res[8];
        unpack8(reinterpret_cast<const uint4*>(xs + r * d)[i], xv);
        if (dres) unpack8(resv[slot][r], res);
        const float4* dyp = reinterpret_cast<const float4*>(dy + r * d + 8 * i);
        const float4 d0 = dyp[0], d1 = dyp[1];
        const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          o[q] = rs * dv[q] * wv[q] - coef * xv[q];
          if (dres) o[q] += res[q];  // residual-stream gradient fused (dh = dres + dx)
          dwacc[slot][q] += dv[q] * xv[q] * rs;
        }
        __stcs(reinterpret_cast<uint4*>(dx + (r0 + r) * d) + i, pack8(o));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int slot = 0; slot < 2; ++slot) {
    const int i = threadIdx.x + slot * kThreads;
    if (i >= nvec) break;
    float4* dst = reinterpret_cast<float4*>(dw_part + static_cast<int64_t>(blockIdx.x) * d + 8 * i);
    dst[0] = make_float4(dwacc[slot][0], dwacc[slot][1], dwacc[slot][2], dwacc[slot][3]);
    dst[1] = make_float4(dwacc[slot][4], dwacc[slot][5], dwacc[slot][6], dwacc[slot][7]);
  }
}

// ---------------------------------------------------------------------------
// Feature-major 8-token variants (tile8.cuh) of the RMSNorm kernels: one
// thread per 8-column vector (blockDim = d / 8), tiles of 8 tokens.  The
// gathered rows are staged as d 16-byte slots, each holding one feature of
// all 8 tokens, so a gather is one 16-byte LDS serving 8 tokens instead of
// eight bank-conflicted 2-byte LDS; 8x8 transposes (PRMT) turn slots back
// into row vectors for coalesced stores.  Same fp32 expressions and
// reduction order as the row-staged kernels at d = 2048.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float block_row_sum(float v, float* red, int r, int nw) {
  // one value per thread for row r -> sum over the block (warp shuffles, then warps in order)
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x % 32 == 0) red[r * 32 + threadIdx.x / 32] = v;
  return v;
}

template <int K>
__global__ void __launch_bounds__(256) rmsnorm_gather_t8_kernel(int64_t T, int d, const __nv_bfloat16* __restrict__ x,
                                                                const float* __restrict__ w, float eps, IdxList outs,
                                                                float* __restrict__ rstd_out) {
  extern __shared__ __align__(16) uint4 slots[];  // d slots
  __shared__ float red[8 * 32];
  __shared__ float rs_s[8];
  const int c = threadIdx.x, nw = blockDim.x / 32;
  float wv[8];
  load_f8(w + 8 * c, wv);
  const int64_t tiles = (T + 7) / 8;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * 8;
    const int nr = static_cast<int>(T - r0 < 8 ? T - r0 : 8);
    uint4 rr[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      rr[r] = r < nr ? __ldcs(reinterpret_cast<const uint4*>(x + (r0 + r) * d) + c) : make_uint4(0, 0, 0, 0);
      float v[8];
      unpack8(rr[r], v);
      float ss = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) ss += v[q] * v[q];
      block_row_sum(ss, red, r, nw);
    }
    __syncthreads();
    if (threadIdx.x < 8) {
      float tot = 0.f;
      for (int k = 0; k < nw; ++k) tot += red[threadIdx.x * 32 + k];
      const float rs = rsqrtf(tot / static_cast<float>(d) + eps);
      rs_s[threadIdx.x] = rs;
      if (threadIdx.x < nr) rstd_out[r0 + threadIdx.x] = rs;
    }
    __syncthreads();
    uint4 yy[8], cc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      float v[8];
      unpack8(rr[r], v);
      const float rs = rs_s[r];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = v[q] * rs * wv[q];
      yy[r] = pack8(v);
    }
    tr8x8(yy, cc);
#pragma unroll
    for (int q = 0; q < 8; ++q) slots[fslot(8 * c + q)] = cc[q];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int id[8];
      load_idx8(outs.idx[k], 8 * c, id);
      uint4 g[8], o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) g[q] = slots[fslot(id[q])];
      tr8x8(g, o);
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(outs.ptr[k]);
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < nr) __stcs(reinterpret_cast<uint4*>(dst + (r0 + r) * d) + c, o[r]);
    }
    __syncthreads();
  }
}

template <int K>
__global__ void __launch_bounds__(256, 2) rmsnorm_gather_bwd_t8_kernel(
    int64_t T, int d, const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
    const float* __restrict__ rstd_in, IdxList dus, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ dw_part) {
  extern __shared__ __align__(16) uint4 slots[];
  __shared__ float red[8 * 32];
  const int c = threadIdx.x, nw = blockDim.x / 32;
  float wv[8], dwacc[8];
  load_f8(w + 8 * c, wv);
#pragma unroll
  for (int q = 0; q < 8; ++q) dwacc[q] = 0.f;
  const int64_t tiles = (T + 7) / 8;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * 8;
    const int nr = static_cast<int>(T - r0 < 8 ? T - r0 : 8);
    float dy[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 8; ++q) dy[r][q] = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {  // dy = sum_k du_k[:, inv_k], k ascending
      const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(dus.ptr[k]);
      uint4 rr[8], cc[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        rr[r] = r < nr ? __ldcs(reinterpret_cast<const uint4*>(src + (r0 + r) * d) + c) : make_uint4(0, 0, 0, 0);
      tr8x8(rr, cc);
#pragma unroll
      for (int q = 0; q < 8; ++q) slots[fslot(8 * c + q)] = cc[q];
      __syncthreads();
      int id[8];
      load_idx8(dus.idx[k], 8 * c, id);
      uint4 g[8], o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) g[q] = slots[fslot(id[q])];
      tr8x8(g, o);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float v[8];
        unpack8(o[r], v);
#pragma unroll
        for (int q = 0; q < 8; ++q) dy[r][q] += v[q];
      }
      __syncthreads();
    }
    float xv[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint4 xr = r < nr ? __ldcs(reinterpret_cast<const uint4*>(x + (r0 + r) * d) + c) : make_uint4(0, 0, 0, 0);
      unpack8(xr, xv[r]);
      float dot = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) dot += dy[r][q] * wv[q] * xv[r][q];
      block_row_sum(dot, red, r, nw);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r >= nr) break;
      float tot = 0.f;
      for (int k = 0; k < nw; ++k) tot += red[r * 32 + k];
      const float rs = rstd_in[r0 + r];
      const float coef = rs * rs * rs * tot / static_cast<float>(d);
      float o[8], res[8];
      if (dres) unpack8(__ldcs(reinterpret_cast<const uint4*>(dres + (r0 + r) * d) + c), res);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        o[q] = rs * dy[r][q] * wv[q] - coef * xv[r][q];
        if (dres) o[q] += res[q];
        dwacc[q] += dy[r][q] * xv[r][q] * rs;
      }
      __stcs(reinterpret_cast<uint4*>(dx + (r0 + r) * d) + c, pack8(o));
    }
    __syncthreads();
  }
  float4* dst = reinterpret_cast<float4*>(dw_part + static_cast<int64_t>(blockIdx.x) * d + 8 * c);
  dst[0] = make_float4(dwacc[0], dwacc[1], dwacc[2], dwacc[3]);
  dst[1] = make_float4(dwacc[4], dwacc[5], dwacc[6], dwacc[7]);
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

// stage 1 of a two-stage column sum: CTA (strip, split) sums its contiguous
// range of rows for 32 columns into mid[split, :] (fixed order)
__global__ void __launch_bounds__(256) colsum_split_kernel(int64_t rows, int64_t d, const float* __restrict__ part,
                                                           float* __restrict__ mid) {
  __shared__ float red[8][33];
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + l;
  const int64_t per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = blockIdx.y * per, r1 = r0 + per < rows ? r0 + per : rows;
  float acc = 0.f;
  if (c < d)
    for (int64_t r = r0 + wp; r < r1; r += 8) acc += part[r * d + c];
  red[wp][l] = acc;
  __syncthreads();
  if (wp == 0 && c < d) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += red[k][l];
    mid[static_cast<int64_t>(blockIdx.y) * d + c] = t;
  }
}

// dw (+)= column sums of the [rows, d] per-CTA partials: two stages so the
// reduction spreads over (d / 32) x kColsumSplits CTAs
int colsum2(int64_t rows, int64_t d, const float* part, float* mid, float* out, int accumulate, cudaStream_t st);

template <int RT, typename IdxT = int32_t>
__global__ void __launch_bounds__(kThreads) swiglu_gather_kernel(
    int64_t T, int f, const __nv_bfloat16* __restrict__ vg, const __nv_bfloat16* __restrict__ vu,
    const IdxT* __restrict__ cg, const IdxT* __restrict__ cu, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* gs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* us = gs + RT * f;
  const int nvec = f / 8;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(gs, vg + r0 * f, nr, f);
    stage_rows(us, vu + r0 * f, nr, f);
    cp_wait_all();
    __syncthreads();
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      int ig[8], iu[8];
      load_idx8(cg, 8 * i, ig);
      load_idx8(cu, 8 * i, iu);
      for (int r = 0; r < nr; ++r) {
        const __nv_bfloat16* grow = gs + r * f;
        const __nv_bfloat16* urow = us + r * f;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float gv = bf(grow[ig[q]]);
          v[q] = gv * sigmoid_f(gv) * bf(urow[iu[q]]);
        }
        __stcs(reinterpret_cast<uint4*>(out + (r0 + r) * f) + i, pack8(v));
      }
    }
    __syncthreads();
  }
}

// dv_g[j] = du[A[j]] * silu'(v_g[j]) * v_u[B[j]] ; dv_u[j] = du[C[j]] * silu(v_g[D[j]])
// on a staged tile of nr rows (gs, us, ds: RT rows each).  C[j] = A[D[j]], so
// dv_u is first formed in gate order (du[A[k]] silu(v_g[k]), no extra gather)
// over the thread's own v_g vector in place, then gathered through D: three
// gathers per element instead of four.
template <int RT, typename IdxT>
__device__ __forceinline__ void swiglu_bwd_tile(int64_t r0, int nr, int f, __nv_bfloat16* gs,
                                                const __nv_bfloat16* us, const __nv_bfloat16* ds,
                                                const IdxT* __restrict__ A, const IdxT* __restrict__ B,
                                                const IdxT* __restrict__ D, __nv_bfloat16* __restrict__ dvg,
                                                __nv_bfloat16* __restrict__ dvu) {
  const int nvec = f / 8;
  for (int i = threadIdx.x; i < nvec; i += kThreads) {
    int ia[8], ib[8];
    load_idx8(A, 8 * i, ia);
    load_idx8(B, 8 * i, ib);
#if POETX_ROW_PROBE == 1  // timing probe: conflict-free identity gathers (results invalid)
#pragma unroll
    for (int q = 0; q < 8; ++q) { ia[q] = (8 * i + q) ^ (ia[q] & 0); ib[q] = (8 * i + q) ^ (ib[q] & 0); }
#endif
    for (int r = 0; r < nr; ++r) {
      const int o = r * f;
      float gself[8], g[8], ug[8];
      uint4* gv = reinterpret_cast<uint4*>(gs + o) + i;
      unpack8(*gv, gself);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float sg = sigmoid_f(gself[q]);
        const float dh = bf(ds[o + ia[q]]);
        g[q] = dh * (sg * (1.f + gself[q] * (1.f - sg))) * bf(us[o + ib[q]]);
        ug[q] = dh * gself[q] * sg;
      }
      __stcs(reinterpret_cast<uint4*>(dvg + (r0 + r) * f) + i, pack8(g));
      *gv = pack8(ug);  // only this thread reads this v_g vector
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nvec; i += kThreads) {
    int id[8];
    load_idx8(D, 8 * i, id);
#if POETX_ROW_PROBE == 1
#pragma unroll
    for (int q = 0; q < 8; ++q) id[q] = (8 * i + q) ^ (id[q] & 0);
#endif
    for (int r = 0; r < nr; ++r) {
      const __nv_bfloat16* row = gs + r * f;
      float u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) u[q] = bf(row[id[q]]);
      __stcs(reinterpret_cast<uint4*>(dvu + (r0 + r) * f) + i, pack8(u));
    }
  }
}

template <int RT, typename IdxT = int32_t>
__global__ void __launch_bounds__(kThreads) swiglu_gather_bwd_kernel(
    int64_t T, int f, const __nv_bfloat16* __restrict__ vg, const __nv_bfloat16* __restrict__ vu,
    const __nv_bfloat16* __restrict__ du, const IdxT* __restrict__ A,
    const IdxT* __restrict__ B, const IdxT* __restrict__ Cc, const IdxT* __restrict__ D,
    __nv_bfloat16* __restrict__ dvg, __nv_bfloat16* __restrict__ dvu) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* gs = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* us = gs + RT * f;
  __nv_bfloat16* ds = us + RT * f;
  (void)Cc;  // C = A o D: dv_u is gathered through D from the gate-order values
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(gs, vg + r0 * f, nr, f);
    stage_rows(us, vu + r0 * f, nr, f);
    stage_rows(ds, du + r0 * f, nr, f);
    cp_wait_all();
    __syncthreads();
    swiglu_bwd_tile<RT, IdxT>(r0, nr, f, gs, us, ds, A, B, D, dvg, dvu);
    __syncthreads();
  }
}

// out = RoPE(z), z[c] = v[inv[c]]; the 8 outputs of a vector lie in one half
// of one head (hd/2 % 8 == 0); hd is a power of two
template <int RT>
__global__ void __launch_bounds__(kThreads) rope_scatter_kernel(
    int64_t T, int S, int H, int hd, const __nv_bfloat16* __restrict__ v,
    const int32_t* __restrict__ inv, const float* __restrict__ cosb, const float* __restrict__ sinb,
    __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(sm);
  const int d = H * hd, half = hd / 2, nvec = d / 8;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(vs, v + r0 * d, nr, d);
    cp_wait_all();
    __syncthreads();
    // one thread: 8 outputs of a head's first half and their 8 partners in
    // the second half -- the 16 gathers feed 16 outputs
    for (int i = threadIdx.x; i < nvec / 2; i += kThreads) {
      const int head = (8 * i) / half, f0 = (8 * i) % half;
      const int c0 = head * hd + f0, c1 = c0 + half;
      int me[8], pa[8];
      load_idx8(inv, c0, me);
      load_idx8(inv, c1, pa);
      for (int r = 0; r < nr; ++r) {
        const int s = static_cast<int>((r0 + r) % S);
        float cs[8], sn[8];
        load_f8(cosb + s * half + f0, cs);
        load_f8(sinb + s * half + f0, sn);
        const __nv_bfloat16* row = vs + r * d;
        float o0[8], o1[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float zm = bf(row[me[q]]), zp = bf(row[pa[q]]);
          o0[q] = zm * cs[q] - zp * sn[q];
          o1[q] = zp * cs[q] + zm * sn[q];
        }
        __nv_bfloat16* orow = out + (r0 + r) * d;
        __stcs(reinterpret_cast<uint4*>(orow + c0), pack8(o0));
        __stcs(reinterpret_cast<uint4*>(orow + c1), pack8(o1));
      }
    }
    __syncthreads();
  }
}

// dv[j] = dz[fwd[j]], dz = RoPE^T(dout) computed on the fly from the staged row
template <int RT>
__global__ void __launch_bounds__(kThreads) rope_scatter_bwd_kernel(
    int64_t T, int S, int H, int hd, const __nv_bfloat16* __restrict__ dout,
    const int32_t* __restrict__ fwd, const float* __restrict__ cosb, const float* __restrict__ sinb,
    __nv_bfloat16* __restrict__ dv) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* os = reinterpret_cast<__nv_bfloat16*>(sm);
  const int d = H * hd, half = hd / 2, nvec = d / 8;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(os, dout + r0 * d, nr, d);
    cp_wait_all();
    __syncthreads();
    // dz = RoPE^T(dout) in place, pairs of contiguous 8-vectors (no gathers)
    for (int i = threadIdx.x; i < nvec / 2; i += kThreads) {
      const int head = (8 * i) / half, f0 = (8 * i) % half;
      const int c0 = head * hd + f0, c1 = c0 + half;
      for (int r = 0; r < nr; ++r) {
        const int s = static_cast<int>((r0 + r) % S);
        float cs[8], sn[8], g0[8], g1[8];
        load_f8(cosb + s * half + f0, cs);
        load_f8(sinb + s * half + f0, sn);
        uint4* p0 = reinterpret_cast<uint4*>(os + r * d + c0);
        uint4* p1 = reinterpret_cast<uint4*>(os + r * d + c1);
        unpack8(*p0, g0);
        unpack8(*p1, g1);
        float d0[8], d1[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          d0[q] = g0[q] * cs[q] + g1[q] * sn[q];
          d1[q] = g1[q] * cs[q] - g0[q] * sn[q];
        }
        *p0 = pack8(d0);
        *p1 = pack8(d1);
      }
    }
    __syncthreads();
    // dv[j] = dz[fwd[j]]: one gather per output
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      int cc[8];
      load_idx8(fwd, 8 * i, cc);
      for (int r = 0; r < nr; ++r) {
        const __nv_bfloat16* row = os + r * d;
        float o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = bf(row[cc[q]]);
        __stcs(reinterpret_cast<uint4*>(dv + (r0 + r) * d) + i, pack8(o));
      }
    }
    __syncthreads();
  }
}

template <int RT>
__global__ void __launch_bounds__(kThreads) scatter_add_kernel(
    int64_t T, int d, const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ v,
    const int32_t* __restrict__ inv, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* vs = reinterpret_cast<__nv_bfloat16*>(sm);
  const int nvec = d / 8;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * RT; r0 < T; r0 += static_cast<int64_t>(gridDim.x) * RT) {
    const int nr = static_cast<int>(T - r0 < RT ? T - r0 : RT);
    stage_rows(vs, v + r0 * d, nr, d);
    cp_wait_all();
    __syncthreads();
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      int id[8];
      load_idx8(inv, 8 * i, id);
      for (int r = 0; r < nr; ++r) {
        float hv[8], o[8];
        unpack8(__ldcs(reinterpret_cast<const uint4*>(h + (r0 + r) * d) + i), hv);
        const __nv_bfloat16* row = vs + r * d;
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = hv[q] + bf(row[id[q]]);
        __stcs(reinterpret_cast<uint4*>(out + (r0 + r) * d) + i, pack8(o));
      }
    }
    __syncthreads();
  }
}


// Token embedding of the trainer (fp32 table, bf16 activations):
//   forward   out[t, :] = bf16(table[tok[t], :])            (gather + cast in one pass)
//   backward  dtable[v, :] += sum over t with tok[t] = v of dh[t, :]
// The backward walks the tokens sorted by id (stable, so positions ascend
// within an id): one warp per run of equal ids sums its rows in fp32 in that
// fixed order and adds the total into the table gradient -- every row is
// written by exactly one warp, no atomics, deterministic.
// Token ids outside [0, V) never address the table: the forward writes a
// NaN row (so the loss turns non-finite and the trainer raises NumericsError,
// as the reference does for a non-finite loss) and the backward skips them.
__global__ void __launch_bounds__(256) embedding_fwd_kernel(int64_t T, int64_t V, int64_t d,
                                                            const int64_t* __restrict__ tok,
                                                            const float* __restrict__ table,
                                                            __nv_bfloat16* __restrict__ out) {
  const int64_t nv = d / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < T * nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / nv, c = i % nv;
    const int64_t id = tok[t];
    float v[8];
    if (id < 0 || id >= V) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __int_as_float(0x7fc00000);
    } else {
      const float4* src = reinterpret_cast<const float4*>(table + id * d) + 2 * c;
      const float4 a = __ldg(src), b = __ldg(src + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    reinterpret_cast<uint4*>(out + t * d)[c] = pack8(v);
  }
}

__global__ void __launch_bounds__(256) embedding_bwd_kernel(int64_t T, int64_t V, int64_t d,
                                                            const int64_t* __restrict__ sorted_tok,
                                                            const int64_t* __restrict__ order,
                                                            const __nv_bfloat16* __restrict__ dh,
                                                            float* __restrict__ dtable) {
  const int lane = threadIdx.x % 32;
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32;
  if (j >= T) return;
  const int64_t id = sorted_tok[j];
  if (id < 0 || id >= V) return;                  // invalid id: no table row (forward wrote NaN)
  if (j > 0 && sorted_tok[j - 1] == id) return;  // not the start of a run
  int64_t end = j + 1;
  while (end < T && sorted_tok[end] == id) ++end;
  for (int64_t c0 = 8 * lane; c0 < d; c0 += 256) {  // 8 columns per lane per chunk
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int64_t k = j; k < end; ++k) {
      float v[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(dh + order[k] * d + c0)), v);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += v[q];
    }
    float4* dst = reinterpret_cast<float4*>(dtable + id * d + c0);
    float4 a = dst[0], b = dst[1];
    a.x += acc[0]; a.y += acc[1]; a.z += acc[2]; a.w += acc[3];
    b.x += acc[4]; b.y += acc[5]; b.z += acc[6]; b.w += acc[7];
    dst[0] = a;
    dst[1] = b;
  }
}

// Cross-entropy over bf16 logits (the trainer's loss head), fused: the
// forward streams each row once with an online max / sum-exp (fp32) and
// keeps (max, sum) per row; the backward streams the row again and writes
// d logits = (softmax - onehot) * g / T straight to bf16 -- no fp32 copy of
// the [T, V] logits in either direction.
__device__ __forceinline__ void ms_combine(float& m, float& s, float m2, float s2) {
  const float M = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - M));
  m = M;
}

__global__ void __launch_bounds__(256) ce_fwd_kernel(int64_t T, int V, const __nv_bfloat16* __restrict__ x,
                                                     const int64_t* __restrict__ tgt, float* __restrict__ loss,
                                                     float* __restrict__ mx, float* __restrict__ se) {
  __shared__ float sm_m[8], sm_s[8];
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32, nv = V / 8;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    const uint4* row = reinterpret_cast<const uint4*>(x + r * V);
    float m = -INFINITY, s = 0.f;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      float v[8];
      unpack8(__ldcs(row + i), v);
      float cm = v[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) cm = fmaxf(cm, v[q]);
      float cs = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) cs += expf(v[q] - cm);
      ms_combine(m, s, cm, cs);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      ms_combine(m, s, m2, s2);
    }
    if (l == 0) { sm_m[wp] = m; sm_s[wp] = s; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float M = sm_m[0], S = sm_s[0];
      for (int k = 1; k < 8; ++k) ms_combine(M, S, sm_m[k], sm_s[k]);
      // targets outside [0, V) (e.g. an ignore_index) are rejected, not
      // ignored: the row's loss is NaN, so the step's loss is non-finite
      const int64_t t = tgt[r];
      const float xt = (t >= 0 && t < V) ? __bfloat162float(x[r * V + t]) : __int_as_float(0x7fc00000);
      loss[r] = (M + logf(S)) - xt;
      mx[r] = M;
      se[r] = S;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) ce_bwd_kernel(int64_t T, int V, const __nv_bfloat16* __restrict__ x,
                                                     const int64_t* __restrict__ tgt, const float* __restrict__ mx,
                                                     const float* __restrict__ se, const float* __restrict__ g0,
                                                     float scale, __nv_bfloat16* __restrict__ grad) {
  const int nv = V / 8;
  const float c = *g0 * scale;
  for (int64_t r = blockIdx.x; r < T; r += gridDim.x) {
    const uint4* row = reinterpret_cast<const uint4*>(x + r * V);
    uint4* out = reinterpret_cast<uint4*>(grad + r * V);
    const float m = mx[r], inv = 1.f / se[r];
    const int64_t t = tgt[r];
    if (t < 0 || t >= V) {  // rejected target (its loss row is NaN): zero gradient row
      for (int i = threadIdx.x; i < nv; i += blockDim.x) __stcs(out + i, make_uint4(0, 0, 0, 0));
      continue;
    }
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      float v[8];
      unpack8(__ldcs(row + i), v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float p = expf(v[q] - m) * inv;
        if (8 * i + q == t) p -= 1.f;
        v[q] = p * c;
      }
      __stcs(out + i, pack8(v));
    }
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
int pick_rt(int64_t bytes_per_row, int64_t default_kb = 48) {
  static int64_t forced = [] {
    const char* e = getenv("POETX_ROW_TILE_KB");
    return static_cast<int64_t>(e ? atoi(e) : 0) * 1024;
  }();
  const int64_t budget = forced > 0 ? forced : default_kb * 1024;
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
#define POETX_RT_DISPATCH_K(rt, KK, KERNEL, ...)              \
  switch (rt) {                                               \
    case 8: { auto k = KERNEL<8, KK>; __VA_ARGS__; break; }   \
    case 4: { auto k = KERNEL<4, KK>; __VA_ARGS__; break; }   \
    case 2: { auto k = KERNEL<2, KK>; __VA_ARGS__; break; }   \
    default: { auto k = KERNEL<1, KK>; __VA_ARGS__; break; }  \
  }
#define POETX_K_DISPATCH(K, rt, KERNEL, ...)                                          \
  switch (K) {                                                                        \
    case 1: POETX_RT_DISPATCH_K(rt, 1, KERNEL, __VA_ARGS__) break;                    \
    case 2: POETX_RT_DISPATCH_K(rt, 2, KERNEL, __VA_ARGS__) break;                    \
    default: POETX_RT_DISPATCH_K(rt, 3, KERNEL, __VA_ARGS__) break;                   \
  }

template <typename K>
void set_smem(K kernel, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

int colsum2(int64_t rows, int64_t d, const float* part, float* mid, float* out, int accumulate, cudaStream_t st) {
  const int splits = static_cast<int>(rows < kColsumSplits ? (rows > 0 ? rows : 1) : kColsumSplits);
  const unsigned strips = static_cast<unsigned>((d + 31) / 32);
  colsum_split_kernel<<<dim3(strips, splits), 256, 0, st>>>(rows, d, part, mid);
  POETX_LAUNCHED("colsum_split");
  colsum_kernel<<<strips, 256, 0, st>>>(splits, d, mid, out, accumulate);
  POETX_LAUNCHED("colsum");
  return POETX_OK;
}

// feature-major 8-token RMSNorm kernels: one thread per 8-column vector, so
// d / 8 must be a whole number of warps within a CTA (env POETX_ROW_T8=0 off)
bool use_t8(int64_t d) {
  static const bool on = [] {
    const char* e = getenv("POETX_ROW_T8");
    return e ? atoi(e) != 0 : true;
  }();
  return on && d % 256 == 0 && d / 8 <= 256;
}
// the backward's T8 variant measured slower (K = 3: 84 vs 74 us at d = 2048;
// 128-register cap, K restagings per tile): opt-in with POETX_ROW_T8_BWD=1
bool use_t8_bwd(int64_t d) {
  static const bool on = [] {
    const char* e = getenv("POETX_ROW_T8_BWD");
    return e && atoi(e) != 0;
  }();
  return on && use_t8(d);
}
unsigned t8_grid(int64_t T, size_t smem) {
  const int64_t tiles = (T + 7) / 8;
  int64_t per_sm = static_cast<int64_t>((228 * 1024) / (smem + 2048));
  if (per_sm > 8) per_sm = 8;
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = 148 * per_sm;
  return static_cast<unsigned>(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
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
  if (use_t8(d)) {
    const size_t tsm = static_cast<size_t>(d) * 16;
    const unsigned grid = t8_grid(T, tsm);
    cudaStream_t st = as_stream(stream);
    switch (K) {
      case 1: set_smem(rmsnorm_gather_t8_kernel<1>, tsm);
              rmsnorm_gather_t8_kernel<1><<<grid, d / 8, tsm, st>>>(T, d, static_cast<const __nv_bfloat16*>(x), w, eps, L, rstd); break;
      case 2: set_smem(rmsnorm_gather_t8_kernel<2>, tsm);
              rmsnorm_gather_t8_kernel<2><<<grid, d / 8, tsm, st>>>(T, d, static_cast<const __nv_bfloat16*>(x), w, eps, L, rstd); break;
      default: set_smem(rmsnorm_gather_t8_kernel<3>, tsm);
               rmsnorm_gather_t8_kernel<3><<<grid, d / 8, tsm, st>>>(T, d, static_cast<const __nv_bfloat16*>(x), w, eps, L, rstd); break;
    }
    POETX_LAUNCHED("rmsnorm_gather_t8");
    return POETX_OK;
  }
  POETX_K_DISPATCH(K, rt, rmsnorm_gather_kernel, set_smem(k, smem);
                   k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(
                       T, d, static_cast<const __nv_bfloat16*>(x), w, eps, L, rstd);)
  POETX_LAUNCHED("rmsnorm_gather");
  return POETX_OK;
}

// the backward re-reads K index maps per tile: larger tiles amortise them
// (measured at Llama-1B shapes: 96 KB tiles 78 us vs 48 KB 86 us)
static int bwd_rt(int64_t d, int K) { return pick_rt(d * 2 * (1 + K) + d * 4, 96); }

size_t poetx_rmsnorm_gather_bwd_workspace_bytes(int64_t T, int64_t d) {
  int rt = bwd_rt(d, 1);  // largest grid over K
  size_t g = row_grid(T, rt);
  const size_t g8 = t8_grid(T, static_cast<size_t>(d) * 16);
  if (g8 > g) g = g8;
  return (g + kColsumSplits) * d * 4 + 256;
}

int poetx_rmsnorm_gather_bwd(int64_t T, int64_t d, const void* x, const float* w, const float* rstd,
                             int K, const int32_t* const* inv, const void* const* du,
                             const void* dres, void* dx, float* dw, int accumulate_dw, void* ws,
                             size_t ws_bytes, void* stream) {
  POETX_REQUIRE(K >= 1 && K <= kMaxK, POETX_ESHAPE, "rmsnorm_gather_bwd: 1..3 inputs");
  POETX_REQUIRE(d <= 16 * kThreads, POETX_ESHAPE, "rmsnorm_gather_bwd: d > %d", 16 * kThreads);
  POETX_REQUIRE(d % 8 == 0, POETX_ESHAPE, "rmsnorm_gather_bwd: d %% 8");
  const int rt = bwd_rt(d, K);
  const size_t smem = rt * d * 2 * (1 + K) + rt * d * 4 + rt * 8 * 4;
  POETX_TRY(check_rows(T, d, smem));
  if (T == 0) return POETX_OK;
  if (use_t8_bwd(d)) {
    const size_t tsm = static_cast<size_t>(d) * 16;
    const unsigned g8 = t8_grid(T, tsm);
    POETX_REQUIRE(ws_bytes >= static_cast<size_t>(g8 + kColsumSplits) * d * 4, POETX_ESHAPE,
                  "rmsnorm_gather_bwd: workspace too small");
    cudaStream_t st = as_stream(stream);
    float* part = static_cast<float*>(ws);
    IdxList L{};
    for (int k = 0; k < K; ++k) { L.idx[k] = inv[k]; L.ptr[k] = const_cast<void*>(du[k]); }
    const auto* xb = static_cast<const __nv_bfloat16*>(x);
    const auto* rb = static_cast<const __nv_bfloat16*>(dres);
    auto* db = static_cast<__nv_bfloat16*>(dx);
    switch (K) {
      case 1: set_smem(rmsnorm_gather_bwd_t8_kernel<1>, tsm);
              rmsnorm_gather_bwd_t8_kernel<1><<<g8, d / 8, tsm, st>>>(T, d, xb, w, rstd, L, rb, db, part); break;
      case 2: set_smem(rmsnorm_gather_bwd_t8_kernel<2>, tsm);
              rmsnorm_gather_bwd_t8_kernel<2><<<g8, d / 8, tsm, st>>>(T, d, xb, w, rstd, L, rb, db, part); break;
      default: set_smem(rmsnorm_gather_bwd_t8_kernel<3>, tsm);
               rmsnorm_gather_bwd_t8_kernel<3><<<g8, d / 8, tsm, st>>>(T, d, xb, w, rstd, L, rb, db, part); break;
    }
    POETX_LAUNCHED("rmsnorm_gather_bwd_t8");
    POETX_TRY(colsum2(g8, d, part, part + static_cast<size_t>(g8) * d, dw, accumulate_dw, st));
    return POETX_OK;
  }
  const unsigned grid = row_grid(T, rt);
  POETX_REQUIRE(ws_bytes >= static_cast<size_t>(grid + kColsumSplits) * d * 4, POETX_ESHAPE,
                "rmsnorm_gather_bwd: workspace too small");
  cudaStream_t st = as_stream(stream);
  float* part = static_cast<float*>(ws);
  IdxList L{};
  for (int k = 0; k < K; ++k) { L.idx[k] = inv[k]; L.ptr[k] = const_cast<void*>(du[k]); }
  POETX_K_DISPATCH(K, rt, rmsnorm_gather_bwd_kernel, set_smem(k, smem);
                   k<<<grid, kThreads, smem, st>>>(T, d, static_cast<const __nv_bfloat16*>(x), w, rstd,
                                                   L, static_cast<const __nv_bfloat16*>(dres),
                                                   static_cast<__nv_bfloat16*>(dx), part);)
  POETX_LAUNCHED("rmsnorm_gather_bwd");
  POETX_TRY(colsum2(grid, d, part, part + static_cast<size_t>(grid) * d, dw, accumulate_dw, st));
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

int poetx_swiglu_gather16(int64_t T, int64_t f, const void* vg, const void* vu, const uint16_t* cg,
                          const uint16_t* cu, void* out, void* stream) {
  POETX_REQUIRE(f <= 65536, POETX_ESHAPE, "swiglu_gather16: f = %lld needs 32-bit maps", (long long)f);
  const int rt = pick_rt(2 * f * 2);
  const size_t smem = rt * 2 * f * 2;
  POETX_TRY(check_rows(T, f, smem));
  if (T == 0) return POETX_OK;
  switch (rt) {
#define POETX_SW16(R)                                                                                          \
  case R: {                                                                                                    \
    auto k = swiglu_gather_kernel<R, uint16_t>;                                                                \
    set_smem(k, smem);                                                                                         \
    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(T, f, static_cast<const __nv_bfloat16*>(vg),    \
                                                             static_cast<const __nv_bfloat16*>(vu), cg, cu,    \
                                                             static_cast<__nv_bfloat16*>(out));                \
    break;                                                                                                     \
  }
    POETX_SW16(8) POETX_SW16(4) POETX_SW16(2) default: POETX_SW16(1)
#undef POETX_SW16
  }
  POETX_LAUNCHED("swiglu_gather16");
  return POETX_OK;
}

int poetx_swiglu_gather_bwd16(int64_t T, int64_t f, const void* vg, const void* vu, const void* du,
                              const uint16_t* A, const uint16_t* B, const uint16_t* Cc, const uint16_t* D,
                              void* dvg, void* dvu, void* stream) {
  POETX_REQUIRE(f <= 65536, POETX_ESHAPE, "swiglu_gather_bwd16: f = %lld needs 32-bit maps", (long long)f);
  const int rt = pick_rt(3 * f * 2);
  const size_t smem = rt * 3 * f * 2;
  POETX_TRY(check_rows(T, f, smem));
  if (T == 0) return POETX_OK;
  switch (rt) {
#define POETX_SWB16(R)                                                                                         \
  case R: {                                                                                                    \
    auto k = swiglu_gather_bwd_kernel<R, uint16_t>;                                                            \
    set_smem(k, smem);                                                                                         \
    k<<<row_grid(T, rt), kThreads, smem, as_stream(stream)>>>(                                                \
        T, f, static_cast<const __nv_bfloat16*>(vg), static_cast<const __nv_bfloat16*>(vu),                   \
        static_cast<const __nv_bfloat16*>(du), A, B, Cc, D, static_cast<__nv_bfloat16*>(dvg),                 \
        static_cast<__nv_bfloat16*>(dvu));                                                                    \
    break;                                                                                                     \
  }
    POETX_SWB16(8) POETX_SWB16(4) POETX_SWB16(2) default: POETX_SWB16(1)
#undef POETX_SWB16
  }
  POETX_LAUNCHED("swiglu_gather_bwd16");
  return POETX_OK;
}

int poetx_rope_scatter(int64_t T, int64_t S, int64_t H, int64_t hd, const void* v,
                       const int32_t* inv, const float* cosb, const float* sinb, void* out,
                       void* stream) {
  POETX_REQUIRE(S > 0 && hd >= 16 && (hd & (hd - 1)) == 0, POETX_ESHAPE,
                "rope_scatter: head_dim must be a power of two >= 16, seq > 0");
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
  POETX_REQUIRE(S > 0 && hd >= 16 && (hd & (hd - 1)) == 0, POETX_ESHAPE,
                "rope_scatter_bwd: head_dim must be a power of two >= 16, seq > 0");
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

int poetx_cross_entropy_fwd(int64_t T, int64_t V, const void* logits, const int64_t* targets, float* loss_rows,
                            float* row_max, float* row_sumexp, void* stream) {
  POETX_REQUIRE(T >= 0 && V > 0 && V % 8 == 0 && V < INT32_MAX, POETX_ESHAPE,
                "cross_entropy: vocab must be a positive multiple of 8, got %lld", (long long)V);
  if (T == 0) return POETX_OK;
  ce_fwd_kernel<<<static_cast<unsigned>(T < 148 * 8 ? T : 148 * 8), 256, 0, as_stream(stream)>>>(
      T, static_cast<int>(V), static_cast<const __nv_bfloat16*>(logits), targets, loss_rows, row_max, row_sumexp);
  POETX_LAUNCHED("cross_entropy_fwd");
  return POETX_OK;
}

int poetx_cross_entropy_bwd(int64_t T, int64_t V, const void* logits, const int64_t* targets, const float* row_max,
                            const float* row_sumexp, const float* dloss, float scale, void* dlogits, void* stream) {
  POETX_REQUIRE(T >= 0 && V > 0 && V % 8 == 0 && V < INT32_MAX, POETX_ESHAPE,
                "cross_entropy: vocab must be a positive multiple of 8, got %lld", (long long)V);
  if (T == 0) return POETX_OK;
  ce_bwd_kernel<<<static_cast<unsigned>(T < 148 * 8 ? T : 148 * 8), 256, 0, as_stream(stream)>>>(
      T, static_cast<int>(V), static_cast<const __nv_bfloat16*>(logits), targets, row_max, row_sumexp, dloss, scale,
      static_cast<__nv_bfloat16*>(dlogits));
  POETX_LAUNCHED("cross_entropy_bwd");
  return POETX_OK;
}

}  // extern "C"

extern "C" {

int poetx_embedding_fwd(int64_t T, int64_t V, int64_t d, const int64_t* tokens, const float* table, void* out,
                        void* stream) {
  POETX_REQUIRE(T >= 0 && V > 0 && d > 0 && d % 8 == 0, POETX_ESHAPE, "embedding_fwd: d %% 8 == 0 required");
  if (T == 0) return POETX_OK;
  const int64_t work = T * (d / 8);
  const unsigned grid = static_cast<unsigned>(work / 256 + 1 < 148 * 16 ? work / 256 + 1 : 148 * 16);
  embedding_fwd_kernel<<<grid, 256, 0, as_stream(stream)>>>(T, V, d, tokens, table, static_cast<__nv_bfloat16*>(out));
  POETX_LAUNCHED("embedding_fwd");
  return POETX_OK;
}

int poetx_embedding_bwd(int64_t T, int64_t V, int64_t d, const int64_t* sorted_tokens, const int64_t* order,
                        const void* dh, float* dtable, void* stream) {
  POETX_REQUIRE(T >= 0 && V > 0 && d > 0 && d % 8 == 0, POETX_ESHAPE, "embedding_bwd: d %% 8 == 0 required");
  if (T == 0) return POETX_OK;
  const unsigned grid = static_cast<unsigned>((T + 7) / 8);
  embedding_bwd_kernel<<<grid, 256, 0, as_stream(stream)>>>(T, V, d, sorted_tokens, order,
                                                            static_cast<const __nv_bfloat16*>(dh), dtable);
  POETX_LAUNCHED("embedding_bwd");
  return POETX_OK;
}

}  // extern "C"
