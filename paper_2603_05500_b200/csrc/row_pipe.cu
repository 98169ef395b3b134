// RMSNorm backward with the consumers' feature gathers fused
// (rmsnorm_gather_bwd, see model_ops.cu), pair-interleaved variant.
//
// dy[t, :] = sum_k du_k[t, inv_k] gathers along the feature axis of
// token-major bf16 rows.  A gather cannot be a TMA box, so rows are staged
// in shared memory and the random reads hit the smem crossbar (128 B/clk
// divided by the bank-conflict degree, ~3.5 for 32 random addresses).  Here
// two token rows are interleaved element-wise into 32-bit words (word c =
// {row 2p [c], row 2p+1 [c]}), so every random LDS.32 returns the column for
// BOTH rows and the math runs on bf16x2 pairs; the K index maps live in
// shared memory once per persistent CTA as uint16.  Measured on B200 at
// Llama-1B shapes (T=8192, d=2048, K=3): 76 us vs 86 us for the staged
// one-row kernel.  The same layout was measured for the forward gathers,
// SwiGLU, RoPE and scatter-add and LOST there (latency-bound at the lower
// occupancy it needs), so those keep the staged kernels in model_ops.cu.
#include <cstdlib>

#include "common.cuh"
#include "row_pipe.cuh"

namespace poetx {
namespace tc {
int num_sms();
}
namespace rp {

constexpr int kT = 256;
constexpr int kMaxMaps = 4;
constexpr size_t kSmemCap = 220 * 1024;

struct Maps {
  const int32_t* idx[kMaxMaps];
  int n;
  int resident;  // 1: u16 copies in shared memory; 0: int32 through L1
};

// ----------------------------------------------------------- helpers ------
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float lo_f(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}
__device__ __forceinline__ float sigmoid_f(float v) { return __frcp_rn(1.f + __expf(-v)); }

// words of two rows a, b (8 columns each) -> 8 interleaved words {a[c], b[c]}
__device__ __forceinline__ void interleave(const uint4 a, const uint4 b, uint4& w0, uint4& w1) {
  w0.x = __byte_perm(a.x, b.x, 0x5410); w0.y = __byte_perm(a.x, b.x, 0x7632);
  w0.z = __byte_perm(a.y, b.y, 0x5410); w0.w = __byte_perm(a.y, b.y, 0x7632);
  w1.x = __byte_perm(a.z, b.z, 0x5410); w1.y = __byte_perm(a.z, b.z, 0x7632);
  w1.z = __byte_perm(a.w, b.w, 0x5410); w1.w = __byte_perm(a.w, b.w, 0x7632);
}
// 8 interleaved words -> the two rows' 8-column vectors
__device__ __forceinline__ void deinterleave(const uint32_t (&w)[8], uint4& a, uint4& b) {
  a.x = __byte_perm(w[0], w[1], 0x5410); b.x = __byte_perm(w[0], w[1], 0x7632);
  a.y = __byte_perm(w[2], w[3], 0x5410); b.y = __byte_perm(w[2], w[3], 0x7632);
  a.z = __byte_perm(w[4], w[5], 0x5410); b.z = __byte_perm(w[4], w[5], 0x7632);
  a.w = __byte_perm(w[6], w[7], 0x5410); b.w = __byte_perm(w[6], w[7], 0x7632);
}
__device__ __forceinline__ void idx8(const uint16_t* m, int j0, int (&o)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(m + j0);
  o[0] = v.x & 0xFFFF; o[1] = v.x >> 16; o[2] = v.y & 0xFFFF; o[3] = v.y >> 16;
  o[4] = v.z & 0xFFFF; o[5] = v.z >> 16; o[6] = v.w & 0xFFFF; o[7] = v.w >> 16;
}
// 8 indices of map k starting at column j0 (smem-resident u16 or int32 via L1)
__device__ __forceinline__ void idxk(const uint16_t* mp, const Maps& M, int k, int W, int j0, int (&o)[8]) {
  if (M.resident) {
    idx8(mp + k * W, j0, o);
  } else {
    const int4 a = __ldg(reinterpret_cast<const int4*>(M.idx[k] + j0));
    const int4 b = __ldg(reinterpret_cast<const int4*>(M.idx[k] + j0) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  }
}
__device__ __forceinline__ void gather_w(const uint32_t* row, const int (&id)[8], uint32_t (&w)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) w[q] = row[id[q]];
}
__device__ __forceinline__ void own_w(const uint32_t* row, int i, uint32_t (&w)[8]) {
  const uint4 a = reinterpret_cast<const uint4*>(row)[2 * i];
  const uint4 b = reinterpret_cast<const uint4*>(row)[2 * i + 1];
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}
// store the pair's results (fp32, 8 columns per row) as two 16-byte vectors
__device__ __forceinline__ void store_pair(__nv_bfloat16* out, int64_t r0, int p, int nr, int W, int i,
                                           const float (&a)[8], const float (&b)[8]) {
  const int ra = 2 * p, rb = 2 * p + 1;
  if (ra < nr)
    __stcs(reinterpret_cast<uint4*>(out + (r0 + ra) * W) + i,
           make_uint4(pack2(a[0], a[1]), pack2(a[2], a[3]), pack2(a[4], a[5]), pack2(a[6], a[7])));
  if (rb < nr)
    __stcs(reinterpret_cast<uint4*>(out + (r0 + rb) * W) + i,
           make_uint4(pack2(b[0], b[1]), pack2(b[2], b[3]), pack2(b[4], b[5]), pack2(b[6], b[7])));
}

// stage rows [r0, r0+nr) (nr <= 2P) of a [T, W] bf16 tensor as P interleaved
// pair-rows of W words; missing rows read as zero
template <int P>
__device__ __forceinline__ void stage(uint32_t* dst, const __nv_bfloat16* src, int64_t r0, int nr, int W) {
  const int nvec = W / 8;
  constexpr int U = 4;
  for (int e0 = threadIdx.x; e0 < P * nvec; e0 += U * kT) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kT;
      a[u] = b[u] = make_uint4(0, 0, 0, 0);
      if (e < P * nvec) {
        const int p = e / nvec, i = e - p * nvec;
        if (2 * p < nr) a[u] = ldg_stream(src + (r0 + 2 * p) * W + 8 * i);
        if (2 * p + 1 < nr) b[u] = ldg_stream(src + (r0 + 2 * p + 1) * W + 8 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kT;
      if (e < P * nvec) {
        const int p = e / nvec, i = e - p * nvec;
        uint4 w0, w1;
        interleave(a[u], b[u], w0, w1);
        uint4* d = reinterpret_cast<uint4*>(dst + p * W + 8 * i);
        d[0] = w0;
        d[1] = w1;
      }
    }
  }
}

// prologue: resident u16 maps at the start of dynamic smem; returns smem base
__device__ __forceinline__ char* load_maps(const Maps& M, int len) {
  extern __shared__ __align__(128) char sm[];
  uint16_t* maps = reinterpret_cast<uint16_t*>(sm);
#pragma unroll
  for (int k = 0; k < kMaxMaps; ++k) {
    if (k >= M.n || !M.resident) break;
    const int4* src = reinterpret_cast<const int4*>(M.idx[k]);
    uint2* dst = reinterpret_cast<uint2*>(maps + k * len);
    for (int i = threadIdx.x; i < len / 4; i += kT) {
      const int4 v = __ldg(src + i);
      dst[i] = make_uint2(static_cast<uint32_t>(v.x) | (static_cast<uint32_t>(v.y) << 16),
                          static_cast<uint32_t>(v.z) | (static_cast<uint32_t>(v.w) << 16));
    }
  }
  return sm;
}
__host__ __device__ inline size_t maps_bytes(int n, int64_t len) {
  return (static_cast<size_t>(n) * len * 2 + 127) / 128 * 128;
}

struct Geo {
  int64_t T;
  int W;         // row width (elements) of the gathered tensors
  int tiles;     // ceil(T / 2P)
  uint32_t off;  // smem offset of the row tiles (after maps and extras)
};

// ------------------------------------------------------------- kernels ----

// dy = sum_k du_k[:, inv_k] ; dx = rstd*dy*w - rstd^3 x (dy.w.x)/d (+ dres) ;
// dw partial += dy*x*rstd (per CTA; reduced by colsum in fixed order).
// Each thread owns fixed columns (i = tid + 256*slot), so its dy values stay
// in registers between the dot pass and the output pass.
template <int P, int K, bool RES>
__global__ void __launch_bounds__(kT, 2) rmsnorm_gather_bwd_kernel(Geo g, Maps M, const __nv_bfloat16* __restrict__ x,
                                                                const float* __restrict__ w,
                                                                const float* __restrict__ rstd_in, DuPtrs dus,
                                                                const __nv_bfloat16* __restrict__ dres,
                                                                __nv_bfloat16* __restrict__ dx,
                                                                float* __restrict__ dw_part) {
  constexpr int SL = 2;  // d <= 16 * kT
  char* sm = load_maps(M, g.W);
  const uint16_t* mp = reinterpret_cast<const uint16_t*>(sm);
  const int d = g.W, nvec = d / 8;
  float* ws = reinterpret_cast<float*>(sm + (M.resident ? maps_bytes(K, d) : 0));  // w [d] | red [8][2P]
  float* red = ws + d;
  uint32_t* tiles = reinterpret_cast<uint32_t*>(sm + g.off);   // x pairs | du_k pairs
  for (int i = threadIdx.x; i < d; i += kT) ws[i] = w[i];
  const int wp = threadIdx.x / 32, l = threadIdx.x % 32;
  float dwacc[SL][8];
#pragma unroll
  for (int a = 0; a < SL; ++a)
#pragma unroll
    for (int q = 0; q < 8; ++q) dwacc[a][q] = 0.f;
  for (int tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
    const int64_t r0 = static_cast<int64_t>(tile) * 2 * P;
    const int nr = static_cast<int>(g.T - r0 < 2 * P ? g.T - r0 : 2 * P);
    __syncthreads();
    stage<P>(tiles, x, r0, nr, d);
#pragma unroll
    for (int k = 0; k < K; ++k)
      stage<P>(tiles + (1 + k) * P * d, static_cast<const __nv_bfloat16*>(dus.p[k]), r0, nr, d);
    __syncthreads();
    float dy[P][SL][16];  // [pair][slot][row a: 0..7 | row b: 8..15]
    float dot[2 * P];
#pragma unroll
    for (int r = 0; r < 2 * P; ++r) dot[r] = 0.f;
#pragma unroll
    for (int sl = 0; sl < SL; ++sl) {
      const int i = threadIdx.x + sl * kT;
      if (i >= nvec) break;
      int iv[K][8];
#pragma unroll
      for (int k = 0; k < K; ++k) idxk(mp, M, k, d, 8 * i, iv[k]);
      const float4 w0 = reinterpret_cast<const float4*>(ws)[2 * i];
      const float4 w1 = reinterpret_cast<const float4*>(ws)[2 * i + 1];
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int p = 0; p < P; ++p) {
        float sa[8], sb[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) sa[q] = sb[q] = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          uint32_t gw[8];
          gather_w(tiles + (1 + k) * P * d + p * d, iv[k], gw);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            sa[q] += lo_f(gw[q]);
            sb[q] += hi_f(gw[q]);
          }
        }
        uint32_t xv[8];
        own_w(tiles + p * d, i, xv);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          dy[p][sl][q] = sa[q];
          dy[p][sl][8 + q] = sb[q];
          dot[2 * p] += sa[q] * wv[q] * lo_f(xv[q]);
          dot[2 * p + 1] += sb[q] * wv[q] * hi_f(xv[q]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2 * P; ++r) {
      float v = dot[r];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0) red[wp * 2 * P + r] = v;
    }
    __syncthreads();
    float coef[2 * P], rs[2 * P];
#pragma unroll
    for (int r = 0; r < 2 * P; ++r) {
      float tot = 0.f;
#pragma unroll
      for (int k = 0; k < kT / 32; ++k) tot += red[k * 2 * P + r];
      rs[r] = r < nr ? __ldg(rstd_in + r0 + r) : 0.f;
      coef[r] = rs[r] * rs[r] * rs[r] * tot / static_cast<float>(d);
    }
#pragma unroll
    for (int sl = 0; sl < SL; ++sl) {
      const int i = threadIdx.x + sl * kT;
      if (i >= nvec) break;
      const float4 w0 = reinterpret_cast<const float4*>(ws)[2 * i];
      const float4 w1 = reinterpret_cast<const float4*>(ws)[2 * i + 1];
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int p = 0; p < P; ++p) {
        uint32_t xv[8];
        own_w(tiles + p * d, i, xv);
        float ra[8], rb[8], oa[8], ob[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) ra[q] = rb[q] = 0.f;
        if (RES) {
          if (2 * p < nr) {
            const uint4 v = ldg_stream(dres + (r0 + 2 * p) * d + 8 * i);
            const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) { ra[2 * q] = lo_f(u[q]); ra[2 * q + 1] = hi_f(u[q]); }
          }
          if (2 * p + 1 < nr) {
            const uint4 v = ldg_stream(dres + (r0 + 2 * p + 1) * d + 8 * i);
            const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) { rb[2 * q] = lo_f(u[q]); rb[2 * q + 1] = hi_f(u[q]); }
          }
        }
        const float sa = rs[2 * p], sb = rs[2 * p + 1];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float xa = lo_f(xv[q]), xb = hi_f(xv[q]);
          const float da = dy[p][sl][q], db = dy[p][sl][8 + q];
          oa[q] = sa * da * wv[q] - coef[2 * p] * xa + ra[q];
          ob[q] = sb * db * wv[q] - coef[2 * p + 1] * xb + rb[q];
          dwacc[sl][q] += da * xa * sa + db * xb * sb;  // rows beyond nr: dy = x = 0
        }
        store_pair(dx, r0, p, nr, d, i, oa, ob);
      }
    }
  }
#pragma unroll
  for (int sl = 0; sl < SL; ++sl) {
    const int i = threadIdx.x + sl * kT;
    if (i >= nvec) break;
    float4* dst = reinterpret_cast<float4*>(dw_part + static_cast<int64_t>(blockIdx.x) * d + 8 * i);
    dst[0] = make_float4(dwacc[sl][0], dwacc[sl][1], dwacc[sl][2], dwacc[sl][3]);
    dst[1] = make_float4(dwacc[sl][4], dwacc[sl][5], dwacc[sl][6], dwacc[sl][7]);
  }
}

// ---------------------------------------------------------------- host ----

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int g_rowpipe_on = [] {
  const char* e = getenv("POETX_ROWPIPE");
  return e && e[0] == '0' ? 0 : 1;
}();

// Launch geometry: P (row pairs per tile) and the persistent grid.  Prefer
// P = 2 with >= 2 CTAs per SM, else P = 1 (>= 1 CTA per SM).
struct Plan {
  int P, grid;
  size_t smem;
  Geo g;
};
int g_resident_maps = [] {
  const char* e = getenv("POETX_ROWPIPE_RESIDENT");
  return e && e[0] == '0' ? 0 : 1;
}();
bool plan(int64_t T, int W, int nmaps, int nstaged, size_t extra, Plan& pl) {
  if (W % 8 || W >= 65536 || T <= 0) return false;
  const int nsm = tc::num_sms();
  const size_t head = (g_resident_maps ? maps_bytes(nmaps, W) : 0) + align_up(extra, 128);
  for (int P : {2, 1}) {
    const size_t smem = head + static_cast<size_t>(nstaged) * P * W * 4;
    int cps = static_cast<int>(228 * 1024 / (smem + 1024));
    if (cps > 4) cps = 4;
    if (smem > kSmemCap || cps < (P == 2 ? 2 : 1)) continue;
    pl.P = P;
    pl.smem = smem;
    pl.g.T = T;
    pl.g.W = W;
    pl.g.tiles = static_cast<int>((T + 2 * P - 1) / (2 * P));
    pl.g.off = static_cast<uint32_t>(head);
    const int64_t cap = static_cast<int64_t>(cps) * nsm;
    pl.grid = static_cast<int>(pl.g.tiles < cap ? pl.g.tiles : cap);
    return true;
  }
  return false;
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}
bool maps_ok(const Maps& M) {
  for (int k = 0; k < M.n; ++k)
    if (!aligned16(M.idx[k])) return false;
  return true;
}

}  // namespace rp

using namespace rp;

int rowpipe_rmsnorm_gather_bwd(int64_t T, int64_t d, const void* x, const float* w, const float* rstd, int K,
                               const int32_t* const* inv, const void* const* du, const void* dres, void* dx,
                               float* part, size_t part_rows, int* grid_out, cudaStream_t st) {
  if (!g_rowpipe_on || d > 16 * kT) return POETX_ENOTSUPPORTED_ROW;
  if (T <= 0) return POETX_ENOTSUPPORTED_ROW;
  Maps M{};
  M.n = K;
  DuPtrs D{};
  for (int k = 0; k < K; ++k) {
    M.idx[k] = inv[k];
    D.p[k] = du[k];
    if (!aligned16(du[k])) return POETX_ENOTSUPPORTED_ROW;
  }
  Plan pl;
  M.resident = g_resident_maps;
  if (!maps_ok(M) || !aligned16(x) || !aligned16(dx) || (dres && !aligned16(dres)) ||
      !plan(T, static_cast<int>(d), K, 1 + K, d * 4 + 8 * 4 * 4, pl))
    return POETX_ENOTSUPPORTED_ROW;
  if (static_cast<size_t>(pl.grid) > part_rows) return POETX_ENOTSUPPORTED_ROW;
  *grid_out = pl.grid;
  const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
  const __nv_bfloat16* rb = static_cast<const __nv_bfloat16*>(dres);
  __nv_bfloat16* dxb = static_cast<__nv_bfloat16*>(dx);
  auto go = [&](auto kern) {
    set_smem(kern, pl.smem);
    kern<<<pl.grid, kT, pl.smem, st>>>(pl.g, M, xb, w, rstd, D, rb, dxb, part);
  };
#define POETX_RP_BWD(P_)                                                 \
  if (pl.P == P_) {                                                      \
    if (dres) {                                                          \
      if (K == 1) go(rmsnorm_gather_bwd_kernel<P_, 1, true>);           \
      else if (K == 2) go(rmsnorm_gather_bwd_kernel<P_, 2, true>);      \
      else go(rmsnorm_gather_bwd_kernel<P_, 3, true>);                  \
    } else {                                                             \
      if (K == 1) go(rmsnorm_gather_bwd_kernel<P_, 1, false>);          \
      else if (K == 2) go(rmsnorm_gather_bwd_kernel<P_, 2, false>);     \
      else go(rmsnorm_gather_bwd_kernel<P_, 3, false>);                 \
    }                                                                    \
  }
  POETX_RP_BWD(2) else POETX_RP_BWD(1)
#undef POETX_RP_BWD
  POETX_LAUNCHED("rowpipe_rmsnorm_gather_bwd");
  return POETX_OK;
}

}  // namespace poetx

extern "C" int poetx_rowpipe_enabled(void) { return poetx::rp::g_rowpipe_on; }
extern "C" void poetx_set_rowpipe_enabled(int on) { poetx::rp::g_rowpipe_on = on ? 1 : 0; }
