// Tensor-core merge (kernel K9; reference
// layer.py:260-273 `_transformed_base`, blockdiag.py:76-97):
//
//   mid = bd(G_R) PM bd(G_P),   tile (s, t) = G_R[s] . PM[sB.., tB..] . G_P[t]
//
// one b x b output tile per CTA (b = 128) or CTA pair (b = 256,
// cta_group::2, CTA c owns rows [128c, 128c + 128) of the tile and holds
// columns [128c, 128c + 128) of every B operand).  The factors stay fp32 in
// meaning: each fp32 operand is split on chip into bf16 hi + lo
// (hi = bf16(x), lo = bf16(x - hi); hi + lo carries ~16 mantissa bits) and
//
//   X = G_R PM      = G_R,hi PM + G_R,lo PM                  (PM is bf16: exact)
//   Y = X G_P      ~= X_hi G_P,hi + X_hi G_P,lo + X_lo G_P,hi
//
// with fp32 accumulation in TMEM (X in accumulator A0, Y in A1); only the
// X_lo G_P,lo term (~2^-18 relative) is dropped.  POET-XQ bases enter as
// int8 codes with per-row scales (quant.py): PM[i, j] = c[i, j] s[i], so the
// scale is folded into the columns of G_R (A' = G_R diag(s), fp32) and the
// codes are exact bf16 B operands.
//
// Operands are written into shared memory by the CTA's threads in the UMMA
// SWIZZLE_128B layouts: A (G_R, X) K-major, B (PM, G_P) MN-major, so every
// global read is a contiguous row segment and no transpose is ever needed.
// The merged tile leaves as bf16 (staged, coalesced 16-byte row stores) or
// fp32 (the requantizing POET-XQ merge).  The composite re-permutation into
// the new premerged order is a separate gather (layer.cu): its column index
// is random at 2-byte granularity, so fusing it into this store would write
// scattered 2-byte sectors.
#include "tc_common.cuh"
#include "tc_gemm.cuh"

namespace poetx {

void* prof_begin(cudaStream_t st);
void prof_end(void* token, const char* name, double flops, cudaStream_t st);

namespace mtc {

using namespace tc;

constexpr int THREADS = 256;

template <int B>
struct Cfg {
  static constexpr bool PAIR = B == 256;
  static constexpr int SLAB = 128 * B * 2;  // 128 rows (A) or 128 columns (B) x B (K), bf16
  static constexpr int SMEM = 3 * SLAB + 1024 + 64;
  static constexpr int TMEM_COLS = 2 * B;
  static constexpr uint32_t IDESC = idesc_bf16(PAIR ? 256 : 128, B, false, true);
};

struct Args {
  int64_t m, n;
  const float* g_r;        // [m/B, B, B] fp32
  const float* g_p;        // [n/B, B, B] fp32
  const __nv_bfloat16* pm; // [m, ldp] bf16 (or null with codes)
  const int8_t* codes;     // [m, ldp] int8 (POET-XQ)
  const float* scales;     // [m] per-row scales (POET-XQ)
  int64_t ldp;
  void* out;               // [m, ldo] bf16 or fp32
  int64_t ldo;
  int out_f32;
};

// K-major SW128 slab of 128 rows: element (r, k), k % 8 == 0
__device__ __forceinline__ uint32_t ka_off(int r, int k) {
  return static_cast<uint32_t>((k >> 6) * 16384 + r * 128 + ((((k & 63) >> 3) ^ (r & 7)) << 4));
}
// MN-major SW128 slab of 128 columns: element (k, c), c % 8 == 0; 64-column
// atoms 8 KB apart, 64-row K chunks 16 KB apart
__device__ __forceinline__ uint32_t mn_off(int k, int c) {
  return static_cast<uint32_t>((k >> 6) * 16384 + (c >> 6) * 8192 + (k & 63) * 128 + ((((c & 63) >> 3) ^ (k & 7)) << 4));
}

__device__ __forceinline__ uint32_t bf16_bits(float x) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(x)));
}
// 8 fp32 values -> bf16 hi / lo units
__device__ __forceinline__ void split8(const float (&v)[8], uint4& hi, uint4& lo) {
  uint32_t h[8], l[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    h[q] = bf16_bits(v[q]);
    l[q] = bf16_bits(v[q] - __uint_as_float(h[q] << 16));
  }
  hi = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
  lo = make_uint4(l[0] | (l[1] << 16), l[2] | (l[3] << 16), l[4] | (l[5] << 16), l[6] | (l[7] << 16));
}

// one 128 x B x B product set into TMEM column offset d (leader thread):
// A K-major slab at a, B MN-major slab at b
template <int B>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint32_t b, bool accumulate) {
#pragma unroll
  for (int kk = 0; kk < B / 16; ++kk) {
    const uint64_t ad = sdesc(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
    const uint64_t bd = sdesc(b + (kk >> 2) * 16384 + (kk & 3) * 2048, 8192, 1024);
    if constexpr (Cfg<B>::PAIR)
      pair::umma2_bf16(d, ad, bd, Cfg<B>::IDESC, (accumulate || kk) ? 1u : 0u);
    else
      umma_bf16(d, ad, bd, Cfg<B>::IDESC, (accumulate || kk) ? 1u : 0u);
  }
}
template <int B>
__device__ __forceinline__ void commit(uint64_t* bar) {
  if constexpr (Cfg<B>::PAIR)
    pair::commit2(bar);
  else
    umma_commit(bar);
}
template <int B>
__device__ __forceinline__ void cta_sync() {
  if constexpr (Cfg<B>::PAIR)
    pair::cluster_sync();
  else
    __syncthreads();
}
// smem operand writes visible to the tensor core, both CTAs of a pair
// arrived, before the leader issues the next products
template <int B>
__device__ __forceinline__ void publish() {
  fence_async_smem();
  fence_before();
  cta_sync<B>();
  fence_after();
}
__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t& phase) {
  mbar_wait(bar, phase);
  phase ^= 1;
  fence_after();
}

// fp32 rows [r0, r0 + 128) x K of a B x B factor block (row-major, optional
// per-column scale) -> K-major hi / lo slabs
template <int B>
__device__ __forceinline__ void load_a(uint8_t* hi, uint8_t* lo, const float* __restrict__ g, int r0,
                                       const float* __restrict__ colscale) {
  for (int e = threadIdx.x; e < 128 * (B / 8); e += THREADS) {
    const int r = e / (B / 8), k = (e % (B / 8)) * 8;
    const float4* src = reinterpret_cast<const float4*>(g + static_cast<int64_t>(r0 + r) * B + k);
    const float4 x0 = __ldg(src), x1 = __ldg(src + 1);
    float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    if (colscale) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] *= __ldg(colscale + k + q);
    }
    uint4 h, l;
    split8(v, h, l);
    *reinterpret_cast<uint4*>(hi + ka_off(r, k)) = h;
    *reinterpret_cast<uint4*>(lo + ka_off(r, k)) = l;
  }
}
// fp32 rows k < B, columns [c0, c0 + 128) of a B x B factor block -> MN-major hi / lo slabs
template <int B>
__device__ __forceinline__ void load_b_f32(uint8_t* hi, uint8_t* lo, const float* __restrict__ g, int c0) {
  for (int e = threadIdx.x; e < B * 16; e += THREADS) {
    const int k = e / 16, c = (e % 16) * 8;
    const float4* src = reinterpret_cast<const float4*>(g + static_cast<int64_t>(k) * B + c0 + c);
    const float4 x0 = __ldg(src), x1 = __ldg(src + 1);
    const float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    uint4 h, l;
    split8(v, h, l);
    *reinterpret_cast<uint4*>(hi + mn_off(k, c)) = h;
    *reinterpret_cast<uint4*>(lo + mn_off(k, c)) = l;
  }
}
// premerged rows [i0, i0 + B), columns [j0, j0 + 128): bf16 as is, or int8 codes (exact in bf16)
template <int B>
__device__ __forceinline__ void load_pm(uint8_t* dst, const Args& a, int64_t i0, int64_t j0) {
  for (int e = threadIdx.x; e < B * 16; e += THREADS) {
    const int k = e / 16, c = (e % 16) * 8;
    const int64_t off = (i0 + k) * a.ldp + j0 + c;
    uint4 u;
    if (a.codes) {
      const uint2 q = __ldg(reinterpret_cast<const uint2*>(a.codes + off));
      const uint32_t w[2] = {q.x, q.y};
      uint32_t h[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) h[x] = bf16_bits(static_cast<float>(static_cast<int8_t>((w[x >> 2] >> (8 * (x & 3))) & 0xFF)));
      u = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
    } else {
      u = __ldg(reinterpret_cast<const uint4*>(a.pm + off));
    }
    *reinterpret_cast<uint4*>(dst + mn_off(k, c)) = u;
  }
}

template <int B>
__global__ void __launch_bounds__(THREADS, 1) merge_tc_kernel(const Args a) {
  using CF = Cfg<B>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* S0 = smem;
  uint8_t* S1 = smem + CF::SLAB;
  uint8_t* S2 = smem + 2 * CF::SLAB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * CF::SLAB);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  const uint32_t rank = CF::PAIR ? pair::cta_rank() : 0;
  const bool issuer = rank == 0 && threadIdx.x == 0;
  const int64_t unit = CF::PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t units = CF::PAIR ? gridDim.x / 2 : gridDim.x;
  const int lo = static_cast<int>(rank) * 128;  // this CTA's rows of the tile / columns of B operands
  const int r = (warp & 3) * 32 + lane;        // TMEM lane = row within this CTA's 128
  const int c_lo = (warp >> 2) * (B / 2);       // this thread's column half

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CF::PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(CF::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(CF::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  fence_before();
  cta_sync<B>();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t A0 = tmem, A1 = tmem + B;
  const uint32_t tl = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t s0 = smem_u32(S0), s1 = smem_u32(S1), s2 = smem_u32(S2);
  uint32_t phase = 0;
  const int64_t nt = a.n / B, tiles = (a.m / B) * nt;

  for (int64_t tile = unit; tile < tiles; tile += units) {
    const int64_t s = tile / nt, t = tile % nt;
    // ---- X = G_R[s] PM_st : S0 <- G_R,hi, S1 <- G_R,lo (this CTA's rows), S2 <- PM (this CTA's columns)
    load_a<B>(S0, S1, a.g_r + s * B * B, lo, a.codes ? a.scales + s * B : nullptr);
    load_pm<B>(S2, a, s * B, t * B + lo);
    publish<B>();
    if (issuer) {
      mma<B>(A0, s0, s2, false);
      mma<B>(A0, s1, s2, true);
      commit<B>(bar);
    }
    wait_mma(bar, phase);
    // ---- Y = X G_P[t] : S0 <- X_hi, S1 <- G_P,hi, S2 <- G_P,lo
    load_b_f32<B>(S1, S2, a.g_p + t * B * B, lo);
#pragma unroll 1
    for (int c = c_lo; c < c_lo + B / 2; c += 32) {
      uint32_t v[32];
      tmem_ld32(A0 + tl + c, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
        u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
        u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
        u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
        *reinterpret_cast<uint4*>(S0 + ka_off(r, c + 8 * q)) = u;
      }
    }
    publish<B>();
    if (issuer) {
      mma<B>(A1, s0, s1, false);
      mma<B>(A1, s0, s2, true);
      commit<B>(bar);
    }
    wait_mma(bar, phase);
    // ---- Y += X_lo G_P,hi : S0 <- X_lo
#pragma unroll 1
    for (int c = c_lo; c < c_lo + B / 2; c += 32) {
      uint32_t v[32];
      tmem_ld32(A0 + tl + c, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float f[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const float xv = __uint_as_float(v[8 * q + x]);
          f[x] = xv - __uint_as_float(bf16_bits(xv) << 16);
        }
        uint4 h, l;
        split8(f, h, l);
        *reinterpret_cast<uint4*>(S0 + ka_off(r, c + 8 * q)) = h;
      }
    }
    publish<B>();
    if (issuer) {
      mma<B>(A1, s0, s1, true);
      commit<B>(bar);
    }
    wait_mma(bar, phase);
    // ---- epilogue: this CTA's 128 rows x B columns of the merged tile
    const int64_t orow0 = s * B + lo;
    if (a.out_f32) {
      float* o = static_cast<float*>(a.out) + (orow0 + r) * a.ldo + t * B;
#pragma unroll 1
      for (int c = c_lo; c < c_lo + B / 2; c += 32) {
        uint32_t v[32];
        tmem_ld32(A1 + tl + c, v);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<uint4*>(o + c + 4 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    } else {
#pragma unroll 1
      for (int c = c_lo; c < c_lo + B / 2; c += 32) {
        uint32_t v[32];
        tmem_ld32(A1 + tl + c, v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
          u.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
          u.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
          u.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
          *reinterpret_cast<uint4*>(S0 + ka_off(r, c + 8 * q)) = u;
        }
      }
      __syncthreads();
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + orow0 * a.ldo + t * B;
      for (int e = threadIdx.x; e < 128 * (B / 8); e += THREADS) {
        const int row = e / (B / 8), u = e % (B / 8);
        *reinterpret_cast<uint4*>(o + row * a.ldo + 8 * u) = *reinterpret_cast<const uint4*>(S0 + ka_off(row, 8 * u));
      }
    }
    // the next tile's operand writes come after every thread's reads of the
    // staging and of TMEM (and, for a pair, the publish barrier orders the peer)
    fence_before();
    __syncthreads();
  }

  fence_before();
  cta_sync<B>();
  fence_after();
  if (warp == 2) {
    if constexpr (CF::PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS) : "memory");
  }
}

template <int B>
int launch(const Args& a, cudaStream_t st) {
  using CF = Cfg<B>;
  auto kern = merge_tc_kernel<B>;
  static bool attr = [&] {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM) == cudaSuccess;
  }();
  POETX_REQUIRE(attr, POETX_ECUDA, "merge_tc: cannot opt in to %d B of shared memory", CF::SMEM);
  const int64_t tiles = (a.m / B) * (a.n / B);
  if (tiles == 0) return POETX_OK;
  const int64_t sms = num_sms();
  const double flops = 5.0 * 2.0 * B * B * static_cast<double>(B) * tiles;  // 2 + 3 products per tile
  void* pf = prof_begin(st);
  if constexpr (CF::PAIR) {
    const int64_t pairs = tiles < sms / 2 ? tiles : sms / 2;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = CF::SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
  } else {
    static int per_sm = [&] {
      int n = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, THREADS, CF::SMEM);
      return n < 1 ? 1 : n;
    }();
    const int64_t ctas = tiles < per_sm * sms ? tiles : per_sm * sms;
    kern<<<static_cast<unsigned>(ctas), THREADS, CF::SMEM, st>>>(a);
  }
  prof_end(pf, "merge_tc", flops, st);
  POETX_LAUNCHED("merge_tc");
  return POETX_OK;
}

}  // namespace mtc
}  // namespace poetx

using namespace poetx;

extern "C" {

int poetx_merge_tc_supported(int64_t b) { return (b == 128 || b == 256) && tc_enabled() ? 1 : 0; }

int poetx_merge_tc(int64_t m, int64_t n, int64_t b, const float* g_r, const float* g_p, const void* pm_bf16,
                   const int8_t* pm_codes, const float* pm_scales, int64_t ldp, void* out, int out_dtype,
                   int64_t ldo, void* stream) {
  POETX_REQUIRE(b == 128 || b == 256, POETX_ESHAPE, "tensor-core merge needs b in {128, 256}, got %lld",
                (long long)b);
  POETX_REQUIRE(m >= 0 && n >= 0 && m % b == 0 && n % b == 0, POETX_ECONFIG,
                "merge_tc: dims (%lld, %lld) must be divisible by block_size %lld", (long long)m, (long long)n,
                (long long)b);
  POETX_REQUIRE(g_r && g_p && out && (pm_bf16 || (pm_codes && pm_scales)), POETX_ESHAPE, "merge_tc: null operand");
  POETX_REQUIRE(out_dtype == POETX_BF16 || out_dtype == POETX_F32, POETX_ESHAPE, "merge_tc: output must be bf16 or f32");
  POETX_REQUIRE(ldp >= n && ldo >= n && ldp % 8 == 0 && ldo % 8 == 0, POETX_ESHAPE,
                "merge_tc: row pitches must be >= n and multiples of 8");
  mtc::Args a{m, n, g_r, g_p, static_cast<const __nv_bfloat16*>(pm_bf16), pm_bf16 ? nullptr : pm_codes,
              pm_bf16 ? nullptr : pm_scales, ldp, out, ldo, out_dtype == POETX_F32 ? 1 : 0};
  cudaStream_t st = as_stream(stream);
  return b == 256 ? mtc::launch<256>(a, st) : mtc::launch<128>(a, st);
}

}  // extern "C"
