// Fused Cayley-Neumann parameterization (k = 3) on tensor cores, one
// kernel per direction (reference cnp.py:71-158).
//
// Every b x b block runs start to finish on chip: the packed fp32
// parameters are unpacked straight into shared memory as the bf16 MMA
// operand, the intermediate products live in TMEM (fp32) and are turned
// back into bf16 operands in shared memory by the CTA's own threads, and
// only the result leaves the SM (G bf16 forward, packed fp32 gradient
// backward).  Nothing is cached between the two directions: the backward
// recomputes Q^2 (one b^3 product) instead of reading a [Q | Q^2] stack.
//
// b = 256: a CTA pair (cta_group::2, M = 256, N = 256); CTA c owns rows
// [128c, 128c + 128) of every b x b operand.  b = 128: one CTA (M = N = 128),
// two CTAs per SM.  Three bf16 operand slabs per CTA (128 rows x b, K-major,
// 128B-swizzled, 64 KB each at b = 256) and two fp32 accumulators in TMEM.
//
// All operands stay CTA-local because every B operand the algebra needs is
// skew or symmetric: an MMA consumes B as rows of B^T, and for Q (skew)
// rows of Q^T are rows of Q negated (the instruction descriptor's negate-B
// bit), for Q^2 (symmetric) they are rows of Q^2.
//
// Forward (G = I + 2(Q + Q^2 + Q^3) + Q^4, cnp.py:109-116):
//   S0 <- 2Q                      (staged packed parameters; x2 is exact)
//   A0  = (2Q)(2Q)                (= 4 Q^2)
//   S1 <- Q^2 = A0 / 4, S0 <- Q^2 - 2Q   (= rows of H^T, H = 2Q + Q^2; in place)
//   A1  = Q^2 H                   (= 2 Q^3 + Q^4)
//   G   = I + (Q^2 - S0) + A0 / 2 + A1
// Two operand slabs, so the NEXT block's packed parameters are bulk-copied
// into the third slab's space while this block computes.
//
// Backward: with N1 = dG, E = N1 - N1^T (skew), F = N1 + N1^T (symmetric),
// the packed gradient g_ij = dQ_ij - dQ_ji (cnp.py:81-86) of the closed-form
// adjoint (cnp.py:136-145) is the upper triangle of
//   P = odd-power part in E - even-power part in F
//     = 2E + 2(E Q^2 + Q E Q + Q^2 E) - 2 V - (V Q^2 + Q^2 V),  V = F Q + Q F
// computed as (7 b^3 products, no transposed operand ever needed):
//   S0 <- Q, S1 <- E, S2 <- F, A1 <- E (fp32, tcgen05.st)
//   A0  = Q E ;  A1 += -(F Q + Q F)                (A1 = E - V)
//   S2 <- Q E ;  S1 <- Z = (A1 + E)/2               (= E - V/2, skew)
//   A0  = Q Q ;  A1 += (Q E) Q
//   S0 <- Q^2
//   A1 += Z Q^2 + Q^2 Z
//   g_ij = 2 A1_ij   (i < j; the fp32 E term rides in the accumulator, so
//                      dG is read from HBM once)
// The next block's packed parameters (and dG) are prefetched into L2 while
// the current block computes.
#include "tc_common.cuh"
#include "tc_gemm.cuh"

namespace poetx {

void* prof_begin(cudaStream_t st);
void prof_end(void* token, const char* name, double flops, cudaStream_t st);

namespace cnpf {

using namespace tc;

constexpr int THREADS = 256;
constexpr uint32_t NEG_A = 1u << 13, NEG_B = 1u << 14;
template <int B>
struct Cfg {
  static constexpr bool PAIR = B == 256;
  static constexpr int SLAB = 128 * B * 2;       // 128 rows x b bf16 (K-major, SW128)
  static constexpr int TILE = 32 * 33 * 4;       // per-warp 32 x 32 fp32 transpose tile
  // forward: two slabs (2Q, Q^2) + the next block's packed staging; backward:
  // three slabs + the per-warp transpose tiles (staging over S1 / S2)
  static constexpr int STG_BYTES = PAIR ? 24512 * 4 : 8128 * 4;  // own packed rows (CTA 0 of a pair is the larger)
  static constexpr int BAR_OFF = (2 * SLAB + STG_BYTES) > (3 * SLAB + 8 * TILE) ? (2 * SLAB + STG_BYTES)
                                                                                : (3 * SLAB + 8 * TILE);
  static constexpr int SMEM = BAR_OFF + 1024 + 64;
  static constexpr int TMEM_COLS = 2 * B;
  static constexpr uint32_t IDESC = idesc_bf16(PAIR ? 256 : 128, B, false, false);
  static constexpr int HALF = B / 2;             // columns per thread in thread-per-row phases
  static constexpr int PITCH = B + 1;            // fp32 staging row pitch (floats): odd, conflict-free
  static_assert(128 * PITCH * 4 <= 3 * SLAB, "fp32 staging must fit in the operand slabs");
};

// byte offset of element (r, j) (j % 8 == 0) in a K-major SW128 slab of 128 rows
__device__ __forceinline__ uint32_t soff(int r, int j) {
  return static_cast<uint32_t>((j >> 6) * 16384 + r * 128 + ((((j & 63) >> 3) ^ (r & 7)) << 4));
}
__device__ __forceinline__ void store32(uint8_t* slab, int r, int j0, const float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16(__float_as_uint(v[8 * q + 0]), __float_as_uint(v[8 * q + 1]));
    u.y = pack_bf16(__float_as_uint(v[8 * q + 2]), __float_as_uint(v[8 * q + 3]));
    u.z = pack_bf16(__float_as_uint(v[8 * q + 4]), __float_as_uint(v[8 * q + 5]));
    u.w = pack_bf16(__float_as_uint(v[8 * q + 6]), __float_as_uint(v[8 * q + 7]));
    *reinterpret_cast<uint4*>(slab + soff(r, j0 + 8 * q)) = u;
  }
}
__device__ __forceinline__ void load32(const uint8_t* slab, int r, int j0, float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = *reinterpret_cast<const uint4*>(slab + soff(r, j0 + 8 * q));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[8 * q + 2 * k] = __uint_as_float(w[k] << 16);
      v[8 * q + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  }
}
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[32]) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
}
// 32 lanes x 32 columns of fp32 into TMEM (this warp's lane quarter)
__device__ __forceinline__ void tmem_st(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// bulk L2 prefetch of a contiguous range (16-byte aligned, multiple of 16 B)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const char* c = static_cast<const char*>(p);
  for (uint32_t o = 0; o < bytes; o += 32768) {
    const uint32_t n = bytes - o < 32768 ? bytes - o : 32768;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(c + o)), "r"(n)
                 : "memory");
  }
}

// Packed strict upper triangle (row-contiguous, cnp.py:66-68): element (i, j),
// i < j, lives at rowp(i) + j with rowp(i) = i*b - i(i+1)/2 - i - 1 (b <= 256,
// so 32-bit offsets).
template <int B>
__device__ __forceinline__ int rowp(int i) {
  return i * B - (i * (i + 1)) / 2 - i - 1;
}

// build-time phase probe (-DPOETX_CNP_TRACE, tools/cnptrace.py): globaltimer
// stamps of thread 0 per phase for the first 5 blocks of every CTA
#ifdef POETX_CNP_TRACE
__device__ unsigned long long g_ctrace[512 * 64];
__device__ __forceinline__ void ctr(int it, int ph) {
  if (threadIdx.x != 0 || it >= 5) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_ctrace[blockIdx.x * 64 + it * 12 + ph] = t;
}
#define CTR(ph) ctr(it, ph)
__device__ unsigned long long g_ctrace_w[512 * 32];  // block 1: per-warp scatter / output start, end
__device__ __forceinline__ void ctrw(int it, int slot) {
  if ((threadIdx.x & 31) != 0 || it != 1) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_ctrace_w[blockIdx.x * 32 + slot] = t;
}
#define CTRW(slot) ctrw(it, slot)
#else
#define CTRW(slot) ((void)(slot))
#define CTR(ph) ((void)(ph))
#endif

// Q rows [lo, lo + 128) of one block from the packed parameters staged in
// shared memory by bulk copies (every global read is a contiguous packed-row
// segment: no per-element loads on the critical path).  Each CTA stages its
// own packed rows [lo, lo + 128) (one contiguous range, 16 B aligned) into
// `stg` and waits on `bar`; a pair's second CTA reads the entries of rows
// j < 128 it needs (-Q[c, j], its "front" columns) from the FIRST CTA's
// staging through distributed shared memory instead of copying 128 separate
// row windows (their bulk-copy requests cost ~4 us per block on warp 0).
template <int B>
struct Stage {
  __device__ static int own_start(int lo) { return rowp<B>(lo) + lo + 1; }
  __device__ static int own_count(int lo) {
    const int hi = lo + 128 < B - 1 ? lo + 128 : B - 1;
    return own_start(hi - 1) + (B - hi) - own_start(lo);  // through the last element of row hi - 1
  }
};
// warp 0: bulk copies of this CTA's packed rows into `stg`, completion on `bar`
template <int B>
__device__ __forceinline__ void stage_issue(float* stg, const float* __restrict__ pk, int lo, uint64_t* bar,
                                            int lane) {
  using ST = Stage<B>;
  const int os = ST::own_start(lo), oc = ST::own_count(lo);
  if (lane == 0) mbar_expect_tx(bar, static_cast<uint32_t>(oc) * 4);
  __syncwarp();
  fence_async_smem();  // earlier generic accesses of the staging area before the async copies
  if (lane == 0) {
    const char* src = reinterpret_cast<const char*>(pk + os);
    for (uint32_t o = 0; o < static_cast<uint32_t>(oc) * 4; o += 32768) {
      const uint32_t n = static_cast<uint32_t>(oc) * 4 - o < 32768 ? static_cast<uint32_t>(oc) * 4 - o : 32768;
      bulk_load_1d(reinterpret_cast<char*>(stg) + o, src + o, n, bar);
    }
  }
}
__device__ __forceinline__ uint32_t dsmem_rank0(uint32_t local) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local));
  return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
// every thread: wait for the staging (and, in a pair, for both CTAs' staging:
// the second CTA reads the first's), then scatter sc * Q into the K-major slab.
// The caller keeps the staging intact until the peer is done (cluster barrier).
template <int B>
__device__ __forceinline__ void stage_scatter(uint8_t* slab, const float* stg, int lo, uint64_t* bar, uint32_t& bph,
                                              int warp, int lane, float sc, int it) {
  (void)it;
  using ST = Stage<B>;
  const float* own = stg;
  const int os = ST::own_start(lo);
  mbar_wait(bar, bph);
  bph ^= 1;
  CTR(10);
  if constexpr (Cfg<B>::PAIR) pair::cluster_sync();  // the first CTA's rows have landed
  // every 32 x 32 tile of this CTA's 128 x b slab: lane = slab row j, its 32
  // values gathered from the staged packed rows, then four 16-byte stores
  // into its own row (4 wavefronts per 512 bytes).  Right of the diagonal a
  // value is Q[j, c] from packed row j (lanes 2-way bank conflicted at
  // most); left of it -Q[c, j] from packed row c (lanes over consecutive j:
  // conflict-free) -- for c < lo from the first CTA's staging (DSMEM); the
  // diagonal tile mixes both and 0, selected arithmetically (per-element
  // branches serialised the warp: 3 us per tile).
  CTRW(2 * warp);
  constexpr int CT = B / 32;
  const uint32_t peer = lo ? dsmem_rank0(smem_u32(stg)) : 0u;  // first CTA's own staging (os = 0 there)
  for (int u = warp; u < 4 * CT; u += 8) {
    // pair: rotate the column tile by half a row of tiles on odd row tiles,
    // so every warp of the second CTA gets two front (DSMEM) tiles, not four
    const int tr = u / CT, tc = Cfg<B>::PAIR ? (u % CT + (tr & 1) * (CT / 2)) % CT : u % CT;
    const int j = lo + 32 * tr + lane, j0 = lo + 32 * tr, c0 = 32 * tc;
    float v[32];
    if (c0 < lo) {
#pragma unroll
      for (int x = 0; x < 32; ++x) v[x] = -sc * ld_dsmem(peer + 4u * static_cast<uint32_t>(rowp<B>(c0 + x) + j));
    } else if (c0 < j0) {
#pragma unroll
      for (int x = 0; x < 32; ++x) v[x] = -sc * own[rowp<B>(c0 + x) - os + j];
    } else if (c0 > j0) {
      const float* row = own + (rowp<B>(j) - os);
#pragma unroll
      for (int x = 0; x < 32; ++x) v[x] = sc * row[c0 + x];
    } else {
      const int rj = rowp<B>(j) - os;
#pragma unroll
      for (int x = 0; x < 32; ++x) {
        const int c = c0 + x;
        // both offsets computed and selected (c == j reads staged element 0;
        // the value is selected away, never multiplied: 0 * NaN of a stale
        // word would poison the diagonal)
        const int il = rowp<B>(c) - os + j, iu = rj + c;
        const float val = own[c > j ? iu : (c < j ? il : 0)];
        v[x] = c > j ? sc * val : (c < j ? -sc * val : 0.f);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      w.x = pack_bf16(__float_as_uint(v[8 * q + 0]), __float_as_uint(v[8 * q + 1]));
      w.y = pack_bf16(__float_as_uint(v[8 * q + 2]), __float_as_uint(v[8 * q + 3]));
      w.z = pack_bf16(__float_as_uint(v[8 * q + 4]), __float_as_uint(v[8 * q + 5]));
      w.w = pack_bf16(__float_as_uint(v[8 * q + 6]), __float_as_uint(v[8 * q + 7]));
      *reinterpret_cast<uint4*>(slab + soff(j - lo, c0 + 8 * q)) = w;
    }
  }
  CTRW(2 * warp + 1);
  CTR(11);
}
template <int B>
__device__ __forceinline__ void unpack_q_staged(uint8_t* slab, float* stg, const float* __restrict__ pk, int lo,
                                                uint64_t* bar, uint32_t& bph, int warp, int lane, int it) {
  if (warp == 0) stage_issue<B>(stg, pk, lo, bar, lane);
  stage_scatter<B>(slab, stg, lo, bar, bph, warp, lane, 1.f, it);
}

// 32 x 32 tile of N1 = dG, one row per lane: a[x] = N1[i0 + lane, j0 + x]
// (read along rows i0.. with lanes over columns, transposed through the
// warp's smem tile) and t[x] = N1[j0 + x, i0 + lane] (lanes over columns of
// row j0 + x: coalesced).
template <int B>
__device__ __forceinline__ void dg_tile_rows(const float* __restrict__ n1, int i0, int j0, int lane, float* tile,
                                             float (&a)[32], float (&t)[32]) {
#pragma unroll
  for (int y = 0; y < 32; ++y) tile[y * 33 + lane] = __ldg(n1 + (i0 + y) * B + j0 + lane);
#pragma unroll
  for (int x = 0; x < 32; ++x) t[x] = __ldg(n1 + (j0 + x) * B + i0 + lane);
  __syncwarp();
#pragma unroll
  for (int x = 0; x < 32; ++x) a[x] = tile[lane * 33 + x];
  __syncwarp();
}

// one b x b x b product into TMEM column offset d (leader thread)
template <int B>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint32_t b, uint32_t flags, bool accumulate) {
  const uint32_t idesc = Cfg<B>::IDESC | flags;
#pragma unroll
  for (int kk = 0; kk < B / 16; ++kk) {
    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
    const uint64_t ad = sdesc(a + off, 16, 1024), bd = sdesc(b + off, 16, 1024);
    if constexpr (Cfg<B>::PAIR)
      pair::umma2_bf16(d, ad, bd, idesc, (accumulate || kk) ? 1u : 0u);
    else
      umma_bf16(d, ad, bd, idesc, (accumulate || kk) ? 1u : 0u);
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

// every thread's smem / TMEM writes are visible to the tensor core, and both
// CTAs of a pair have arrived, before the leader issues the next products
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


template <int B, bool FWD>
__global__ void __launch_bounds__(THREADS, 1)
    cnp_fused_kernel(const __grid_constant__ CUtensorMap gmap, int64_t nb, const float* __restrict__ packed,
                     const float* __restrict__ dg, __nv_bfloat16* __restrict__ g16, float* __restrict__ g32,
                     float* __restrict__ dpacked, int accumulate) {
  using CF = Cfg<B>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by offsetting the shared array itself (keeps the
  // pointers in the shared address space: STS/LDS, not generic accesses)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* S0 = smem;
  uint8_t* S1 = smem + CF::SLAB;
  uint8_t* S2 = smem + 2 * CF::SLAB;
  float* stage = reinterpret_cast<float*>(smem);  // fp32 staging over the slabs (final phase)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* tile = reinterpret_cast<float*>(smem + 3 * CF::SLAB) + warp * (32 * 33);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + CF::BAR_OFF);
  uint64_t* sbar = bar + 1;  // packed-parameter staging (bulk copies)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);

  const uint32_t rank = CF::PAIR ? pair::cta_rank() : 0;
  const bool issuer = rank == 0 && threadIdx.x == 0;
  const int64_t unit = CF::PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t units = CF::PAIR ? gridDim.x / 2 : gridDim.x;
  const int lo = static_cast<int>(rank) * 128;     // this CTA's rows of the b x b block
  const int r = (warp & 3) * 32 + lane;           // TMEM lane = row within this CTA's 128
  const int c_lo = (warp >> 2) * CF::HALF;         // this thread's column half

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(sbar, 1);
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
  const uint32_t A0 = tmem, A1 = tmem + B;                           // accumulators (columns)
  const uint32_t tl = static_cast<uint32_t>((warp & 3) * 32) << 16;  // this warp's TMEM lanes
  const uint32_t s0 = smem_u32(S0), s1 = smem_u32(S1), s2 = smem_u32(S2);
  uint32_t phase = 0, sphase = 0;
  constexpr int64_t PAIRS = static_cast<int64_t>(B) * (B - 1) / 2;
  // packed staging: backward over S1 / S2 (free at unpack time); forward
  // behind S0 / S1, filled for the NEXT block while this one computes
  float* stg = reinterpret_cast<float*>(FWD ? S2 : S1);
  static_assert(CF::STG_BYTES <= 2 * CF::SLAB && 24512 * 4 <= CF::STG_BYTES + (B == 256 ? 0 : 1 << 30),
                "packed staging must fit");
  if constexpr (FWD) {
    if (warp == 0 && unit < nb) stage_issue<B>(stg, packed + unit * PAIRS, lo, sbar, lane);
  }

  int it = -1;
  for (int64_t s = unit; s < nb; s += units) {
    ++it;
    (void)it;
    CTR(0);
    const float* pk = packed + s * PAIRS;
    // the forward already stages the next block's parameters during this one:
    // its L2 prefetch runs one block further ahead
    const int64_t pre = FWD ? s + 2 * units : s + units;
    if (threadIdx.x == 0 && pre < nb) {
      // upcoming inputs into L2 while this block computes (each CTA of a pair
      // fetches half): their staging / loads then wait on L2, not DRAM, latency
      constexpr uint32_t PB = static_cast<uint32_t>(PAIRS) * 4, HB = PB / 32 * 16;
      const char* nx = reinterpret_cast<const char*>(packed + pre * PAIRS);
      if (CF::PAIR)
        prefetch_l2(nx + rank * HB, rank ? PB - HB : HB);
      else
        prefetch_l2(nx, PB);
      if (!FWD) {
        constexpr uint32_t DB = static_cast<uint32_t>(B) * B * 4 / (CF::PAIR ? 2 : 1);
        prefetch_l2(reinterpret_cast<const char*>(dg + (s + units) * B * B) + rank * DB, DB);
      }
    }
    if constexpr (FWD) {
      // ---- S0 <- 2Q (the staged packed parameters, scaled exactly by 2)
      stage_scatter<B>(S0, stg, lo, sbar, sphase, warp, lane, 2.f, it);
      // S1 is rewritten after the first product: the previous block's G
      // stores (TMA, from S1) must have read it
      if (g16 && threadIdx.x == 0) bulk_wait_read<0>();
      __syncthreads();  // the staging is consumed: the next block's copies may land
      CTR(1);
      publish<B>();
      if (issuer) {
        mma<B>(A0, s0, s0, NEG_B, false);  // 4 Q^2 = (2Q) (-(2Q))^T
        commit<B>(bar);
      }
      if (warp == 0 && s + units < nb) stage_issue<B>(stg, packed + (s + units) * PAIRS, lo, sbar, lane);
      wait_mma(bar, phase);
      CTR(2);
      // ---- S1 <- Q^2 = A0 / 4 (exact scaling) ; S0 <- Q^2 - 2Q (rows of H^T,
      // H = 2Q + Q^2), in place over this thread's own 2Q row chunk
#pragma unroll 1
      for (int c = c_lo; c < c_lo + CF::HALF; c += 32) {
        float q2[32], tq[32];
        tmem_ld(A0 + tl + c, q2);
        load32(S0, r, c, tq);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          q2[k] *= 0.25f;
          tq[k] = q2[k] - tq[k];
        }
        store32(S1, r, c, q2);
        store32(S0, r, c, tq);
      }
      CTR(3);
      publish<B>();
      if (issuer) {
        mma<B>(A1, s1, s0, 0, false);  // Q^2 H = 2 Q^3 + Q^4
        commit<B>(bar);
      }
      wait_mma(bar, phase);
      CTR(4);
      // ---- G = I + 2Q + 2Q^2 + (2 Q^3 + Q^4), staged bf16 in S1 (its rows are
      // this thread's); 2Q = Q^2 - bf16(Q^2 - 2Q), within 2^-8 |Q| of exact
      const int64_t grow = (s * B + lo + r) * B;
#pragma unroll 1
      for (int c = c_lo; c < c_lo + CF::HALF; c += 32) {
        float h[32], q2[32], p[32];
        load32(S0, r, c, h);       // Q^2 - 2Q (bf16)
        tmem_ld(A0 + tl + c, q2);  // 4 Q^2 (fp32)
        tmem_ld(A1 + tl + c, p);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float qq = 0.25f * q2[k];
          p[k] = (qq - h[k]) + 2.f * qq + p[k];
          if (c + k == lo + r) p[k] += 1.f;
        }
        if (g16) store32(S1, r, c, p);
        if (g32) {
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            *reinterpret_cast<float4*>(g32 + grow + c + 4 * q4) =
                make_float4(p[4 * q4], p[4 * q4 + 1], p[4 * q4 + 2], p[4 * q4 + 3]);
        }
      }
      CTR(5);
      if (g16) {
        // the bf16 rows of G leave through TMA stores straight from the
        // swizzled slab (one 64-column x 128-row box per 128-byte atom column);
        // they drain while the next block unpacks and multiplies
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
          for (int k = 0; k < B / 64; ++k)
            tma_store_2d(&gmap, S1 + k * 16384, 64 * k, static_cast<int>(s * B + lo));
          bulk_commit();
        }
      }
      // the next block's unpack overwrites S0 / S1 only after this CTA's
      // threads passed the publish barrier, i.e. after these reads
      __syncthreads();
      CTR(6);
    } else {
      const float* n1 = dg + s * static_cast<int64_t>(B) * B;
      // ---- S0 <- Q ; S1 <- E = N1 - N1^T ; S2 <- F = N1 + N1^T ; A1 <- E (fp32)
      // (warp w owns TMEM lanes [32 (w & 3), +32): its tiles are that row group)
      unpack_q_staged<B>(S0, stg, pk, lo, sbar, sphase, warp, lane, it);
      cta_sync<B>();  // the staging (S1 / S2; the peer reads the first CTA's) is read before E / F overwrite it
      CTR(1);
      for (int k = 0; k < B / 64; ++k) {
        const int i0 = lo + (warp & 3) * 32, j0 = ((warp >> 2) * (B / 64) + k) * 32;
        float a[32], t[32];
        dg_tile_rows<B>(n1, i0, j0, lane, tile, a, t);
#pragma unroll
        for (int x = 0; x < 32; ++x) {
          const float e = a[x] - t[x];
          a[x] += t[x];
          t[x] = e;
        }
        tmem_st(A1 + tl + j0, t);            // E, the fp32 start of the accumulator
        store32(S1, i0 - lo + lane, j0, t);  // E
        store32(S2, i0 - lo + lane, j0, a);  // F
      }
      tmem_st_wait();
      CTR(2);
      publish<B>();
      if (issuer) {
        mma<B>(A0, s0, s1, NEG_B, false);  // Q E = S0 (-S1)^T          (E = -E^T)
        mma<B>(A1, s2, s0, 0, true);       // E - (F Q) = S2 S0^T       (Q = -S0^T)
        mma<B>(A1, s0, s2, NEG_A, true);   // -(Q F) = (-S0) S2^T       (F = F^T)
        commit<B>(bar);
      }
      wait_mma(bar, phase);
      CTR(3);
      // ---- S2 <- Q E ; S1 <- Z = E - V/2 = (A1 + E) / 2   (A1 = E - V)
#pragma unroll 1
      for (int c = c_lo; c < c_lo + CF::HALF; c += 32) {
        float v[32], e[32];
        tmem_ld(A0 + tl + c, v);
        store32(S2, r, c, v);
        tmem_ld(A1 + tl + c, v);
        load32(S1, r, c, e);
#pragma unroll
        for (int k = 0; k < 32; ++k) e[k] = 0.5f * (e[k] + v[k]);
        store32(S1, r, c, e);
      }
      CTR(4);
      publish<B>();
      if (issuer) {
        mma<B>(A0, s0, s0, NEG_B, false);  // Q Q
        mma<B>(A1, s2, s0, NEG_B, true);   // += (Q E) Q
        commit<B>(bar);
      }
      wait_mma(bar, phase);
      CTR(5);
      // ---- S0 <- Q^2
#pragma unroll 1
      for (int c = c_lo; c < c_lo + CF::HALF; c += 32) {
        float v[32];
        tmem_ld(A0 + tl + c, v);
        store32(S0, r, c, v);
      }
      CTR(6);
      publish<B>();
      if (issuer) {
        mma<B>(A1, s1, s0, 0, true);      // += Z Q^2        (Q^2 = (Q^2)^T)
        mma<B>(A1, s0, s1, NEG_B, true);  // += Q^2 Z = Q^2 (-S1)^T
        commit<B>(bar);
      }
      wait_mma(bar, phase);
      CTR(7);
      // ---- stage A1 = E + R (fp32, thread per row, odd pitch: conflict-free
      // for row and column reads) over the slabs, then per 32 x 32 tile of the
      // upper triangle g_ij = 2 A1_ij written as coalesced runs of packed rows.
      // P = A1 is skew-symmetric (every term is: E, V, E Q^2 + Q E Q + Q^2 E,
      // V Q^2 + Q^2 V), so g_ij = -2 A1_ji too: each CTA of a pair writes the
      // upper tiles of its own diagonal quadrant and half of the off-diagonal
      // quadrant -- CTA 0 from its rows i < 128, CTA 1 from its rows j >= 128
      // transposed -- all from its own staging (no peer reads, balanced).
#pragma unroll 1
      for (int c = c_lo; c < c_lo + CF::HALF; c += 32) {
        float v[32];
        tmem_ld(A1 + tl + c, v);
#pragma unroll
        for (int k = 0; k < 32; ++k) stage[r * CF::PITCH + c + k] = v[k];
      }
      __syncthreads();
      CTR(8);
      float* out = dpacked + s * PAIRS;
      CTRW(16 + 2 * warp);
      {
        constexpr int NT = B / 32, QT = 4;  // tiles per side; per 128-row quadrant
        const int q0 = lo / 32;             // this CTA's diagonal quadrant
        int k = 0;
        for (int ta = 0; ta < NT; ++ta) {
          for (int tb = ta; tb < NT; ++tb) {
            const bool diag = ta >= q0 && tb < q0 + QT;                       // own quadrant
            const bool off = CF::PAIR && ta < QT && tb >= QT && ((ta + tb) & 1) == static_cast<int>(rank);
            if (!diag && !off) continue;
            if (k++ % 8 != warp) continue;
            const int i0 = 32 * ta, j0 = 32 * tb, j = j0 + lane;
            const bool trans = off && rank == 1;  // g_ij = -2 P_ji from own row j
            // 16 rows at a time: every shared load (and, accumulating, every
            // global read) of the group in flight before the stores
#pragma unroll 1
            for (int y0 = 0; y0 < 32; y0 += 16) {
              float gv[16];
              // unconditional loads, arithmetic selects (a load under a
              // per-lane condition compiles to a divergent branch per row)
              const float sg = trans ? -2.f : 2.f;
#pragma unroll
              for (int y = 0; y < 16; ++y) {
                const int i = i0 + y0 + y;
#if POETX_CNP_OUT_PROBE == 3
                const float val = static_cast<float>(i * j);  // probe: no staging loads
#else
                const float val = stage[trans ? (j - lo) * CF::PITCH + i : (i - lo) * CF::PITCH + j];
#endif
                gv[y] = j > i ? sg * val : 0.f;
              }
              if (accumulate) {
#pragma unroll
                for (int y = 0; y < 16; ++y) {
                  const int i = i0 + y0 + y;
                  if (j > i) gv[y] += out[rowp<B>(i) + j];
                }
              }
#pragma unroll
              for (int y = 0; y < 16; ++y) {
                const int i = i0 + y0 + y;
#if POETX_CNP_OUT_PROBE == 1
                if (j > i && gv[y] == 12345.f) out[rowp<B>(i) + j] = gv[y];  // probe: stores compiled out
#elif POETX_CNP_OUT_PROBE == 2
                out[((i * 8 + (j0 >> 5)) * 32 + lane) & 16383] = gv[y];  // probe: aligned 128-byte rows
#else
                if (j > i) out[rowp<B>(i) + j] = gv[y];
#endif
              }
            }
          }
        }
      }
      CTRW(17 + 2 * warp);
      // the next block's unpack overwrites this CTA's staging only after every
      // warp is done reading it (the peer never reads it)
      __syncthreads();
      CTR(9);
    }
  }

  if (FWD && g16 && threadIdx.x == 0) bulk_wait<0>();  // G stores done with the slab
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

template <int B, bool FWD>
int launch(int64_t nb, const float* packed, const float* dg, __nv_bfloat16* g16, float* g32, float* dpacked,
           int accumulate, cudaStream_t st) {
  using CF = Cfg<B>;
  auto kern = cnp_fused_kernel<B, FWD>;
  static bool attr = [&] {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM) == cudaSuccess;
  }();
  POETX_REQUIRE(attr, POETX_ECUDA, "cnp_fused: cannot opt in to %d B of shared memory", CF::SMEM);
  const int64_t sms = num_sms();
  CUtensorMap gmap{};
  if (FWD && g16)  // G as [nb * B rows, B cols] bf16, 64 x 128 boxes, 128-byte swizzle (the slab layout)
    POETX_TRY(make_map(&gmap, g16, B, static_cast<uint64_t>(nb) * B, B, 64, 128));
  unsigned grid;
  if constexpr (CF::PAIR) {
    const int64_t pairs = nb < sms / 2 ? nb : sms / 2;
    grid = static_cast<unsigned>(2 * pairs);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = CF::SMEM;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* pf = prof_begin(st);
    cudaLaunchKernelEx(&cfg, kern, gmap, nb, packed, dg, g16, g32, dpacked, accumulate);
    prof_end(pf, FWD ? "cnp_fused_fwd" : "cnp_fused_bwd", (FWD ? 2.0 : 7.0) * 2.0 * B * B * B * nb, st);
  } else {
    static int per_sm = [&] {
      int n = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, THREADS, CF::SMEM);
      return n < 1 ? 1 : n;
    }();
    const int64_t ctas = nb < per_sm * sms ? nb : per_sm * sms;
    grid = static_cast<unsigned>(ctas);
    void* pf = prof_begin(st);
    kern<<<grid, THREADS, CF::SMEM, st>>>(gmap, nb, packed, dg, g16, g32, dpacked, accumulate);
    prof_end(pf, FWD ? "cnp_fused_fwd" : "cnp_fused_bwd", (FWD ? 2.0 : 7.0) * 2.0 * B * B * B * nb, st);
  }
  POETX_LAUNCHED(FWD ? "cnp_fused_fwd" : "cnp_fused_bwd");
  return POETX_OK;
}

}  // namespace cnpf
}  // namespace poetx

using namespace poetx;

extern "C" {

int poetx_cnp_fused_supported(int64_t b) { return (b == 128 || b == 256) && tc_enabled() ? 1 : 0; }

int poetx_cnp_forward_fused(int64_t nb, int64_t b, const float* packed, void* g_bf16, float* g_f32, void* stream) {
  POETX_REQUIRE(b == 128 || b == 256, POETX_ESHAPE, "fused tensor-core CNP needs b in {128, 256}, got %lld",
                (long long)b);
  POETX_REQUIRE(nb >= 0 && packed && (g_bf16 || g_f32), POETX_ESHAPE, "cnp_forward_fused: null operand");
  if (nb == 0) return POETX_OK;
  auto* g16 = static_cast<__nv_bfloat16*>(g_bf16);
  cudaStream_t st = as_stream(stream);
  return b == 256 ? cnpf::launch<256, true>(nb, packed, nullptr, g16, g_f32, nullptr, 0, st)
                  : cnpf::launch<128, true>(nb, packed, nullptr, g16, g_f32, nullptr, 0, st);
}

int poetx_cnp_backward_fused(int64_t nb, int64_t b, const float* packed, const float* dg, float* dpacked,
                             int accumulate, void* stream) {
  POETX_REQUIRE(b == 128 || b == 256, POETX_ESHAPE, "fused tensor-core CNP needs b in {128, 256}, got %lld",
                (long long)b);
  POETX_REQUIRE(nb >= 0 && packed && dg && dpacked, POETX_ESHAPE, "cnp_backward_fused: null operand");
  if (nb == 0) return POETX_OK;
  cudaStream_t st = as_stream(stream);
  return b == 256 ? cnpf::launch<256, false>(nb, packed, dg, nullptr, nullptr, dpacked, accumulate, st)
                  : cnpf::launch<128, false>(nb, packed, dg, nullptr, nullptr, dpacked, accumulate, st);
}

}  // extern "C"

#ifdef POETX_CNP_TRACE
extern "C" int poetx_cnp_trace_copy(unsigned long long* host, int n) {
  if (n > 512 * 64) n = 512 * 64;
  return static_cast<int>(cudaMemcpyFromSymbol(host, poetx::cnpf::g_ctrace, n * sizeof(unsigned long long)));
}
extern "C" int poetx_cnp_trace_copy_w(unsigned long long* host, int n) {
  if (n > 512 * 32) n = 512 * 32;
  return static_cast<int>(cudaMemcpyFromSymbol(host, poetx::cnpf::g_ctrace_w, n * sizeof(unsigned long long)));
}
extern "C" int poetx_cnp_trace_reset() {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, poetx::cnpf::g_ctrace) != cudaSuccess) return 1;
  return static_cast<int>(cudaMemset(p, 0, sizeof(poetx::cnpf::g_ctrace)));
}
#endif
