// tcgen05 / TMEM / TMA tensor-core kernels for the BF16 path (sm_100a).
//
// One warp-specialised, persistent kernel serves every tensor-core product
// on the POET-X path as a *grouped* GEMM
//
//   for g in groups, s in k-splits:   C[g, s][M, N] = A[g][M, K_s] . B[g][K_s, N]
//
// with BF16 operands addressed through 2-D TMA tensor maps (each group adds
// a fixed coordinate offset, so block-diagonal segments, stacks of b x b
// blocks and split-K slices are all views of one tensor, never copies),
// either operand K-major or MN-major (a transposed operand is just the
// other major in the UMMA instruction descriptor), and FP32 accumulation
// in TMEM written out as BF16 or FP32:
//
//   mm2 t = a PM / adjoint da = dt PM^T    (layer.py:222, 249)   1 group
//   apply_to_features y_s = x_s G[s]       (blockdiag.py:58-73)  nb groups
//   segmented_outer dG[s] = x_s^T y_s      (blockdiag.py:100-121) nb groups x splits
//   CNP products Q^2, Q^2 Q, ...           (cnp.py:99-145)       nb groups
//
// Roles (one CTA per SM, 256 threads):
//   warp 0      TMA producer: STAGES-deep ring of {A 128x64, B BNx64}
//               SWIZZLE_128B tiles, mbarrier full/empty handshake;
//   warp 1      MMA issuer: one lane issues tcgen05.mma (M=128, N=BN, K=16)
//               into a double-buffered TMEM accumulator; tcgen05.commit
//               releases smem stages / publishes finished accumulators;
//   warp 2      TMEM allocator;
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> BF16/FP32 -> global, then
//               release the accumulator (next tile's MMAs overlap the store).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tc_common.cuh"
#include "tc_gemm.cuh"

namespace poetx {

void* prof_begin(cudaStream_t st);
void prof_end(void* token, const char* name, double flops, cudaStream_t st);

static int g_tc_on = 1;
bool tc_enabled() { return g_tc_on != 0; }

namespace tc {

constexpr int THREADS = 256;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB

// MS = number of 128-row M sub-tiles per CTA tile sharing each B stage
// (MS = 2 halves the B operand traffic of tall-K, small-N problems such as
// the segmented outer product).
template <int BN, int MS> struct Cfg {
  static constexpr int A_BYTES_T = MS * A_BYTES;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES_T + B_BYTES;
  static constexpr int STAGES_RAW = (192 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int EPI_BYTES = 4 * 2 * 32 * 128;  // per warp: 2 x (32 rows x 128 B)
  static constexpr int ACC_COLS = MS * BN;                 // one accumulator (all sub-tiles)
  static constexpr int NACC = (2 * ACC_COLS <= 512) ? 2 : 1;
  static constexpr int TMEM_NEED = NACC * ACC_COLS;
  static constexpr int TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128
                                 : TMEM_NEED <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

struct Args {
  int M, N, K;             // per group; K is split into `splits` chunks of kps
  int groups, splits, kps;
  int m_tiles, n_tiles;
  int a_g0, a_g1, b_g0, b_g1;  // per-group TMA coordinate offsets (c0, c1)
  void* C;
  int64_t ldc, c_goff, c_soff;  // element strides: row, group, split
  int out_f32;
  int accumulate;  // fp32 output only: C += alpha * AB
  float alpha;
  int tma_epi;     // 1: epilogue through smem staging + TMA bulk store (reduce-add if accumulate)
  int64_t c_row0;  // row of C (in map_c) where group 0 / split 0 starts ... per-group/split rows:
  int64_t c_grow, c_srow;
  const float* bscale;  // int8 B (pair kernel Q8): fp32 scale per row of the B tensor view
};

// ------------------------------------------------------------------ kernel --
template <int BN, bool A_MN, bool B_MN, int MS>
__global__ void __launch_bounds__(THREADS, 1)
    tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
              const __grid_constant__ CUtensorMap map_c, Args args) {
  using CF = Cfg<BN, MS>;
  constexpr int STAGES = CF::STAGES, NACC = CF::NACC, TM = BM * MS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = /* 1024-byte aligned, kept in the shared address space (STS/LDS) */ smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi = smem + STAGES * CF::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + CF::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [NACC]
  uint64_t* tempty = tfull + 2;      // [NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_per_split = args.m_tiles * args.n_tiles;
  const int num_tiles = tiles_per_split * args.splits * args.groups;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](int tile, int& g, int& s, int& m0, int& n0, int& kb0, int& kbn) {
    g = tile / (tiles_per_split * args.splits);
    int r = tile % (tiles_per_split * args.splits);
    s = r / tiles_per_split;
    r %= tiles_per_split;
    m0 = (r / args.n_tiles) * TM;
    n0 = (r % args.n_tiles) * BN;
    int k0 = s * args.kps;
    int k1 = k0 + args.kps < args.K ? k0 + args.kps : args.K;
    kb0 = k0 / BK;
    kbn = (k1 - k0 + BK - 1) / BK;
  };

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int g, s, m0, n0, kb0, kbn;
        decode(tile, g, s, m0, n0, kb0, kbn);
        const int ag0 = args.a_g0 * g, ag1 = args.a_g1 * g;
        const int bg0 = args.b_g0 * g, bg1 = args.b_g1 * g;
        for (int kb = kb0; kb < kb0 + kbn; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * CF::STAGE_BYTES;
          uint8_t* sb = sa + CF::A_BYTES_T;
          const int k = kb * BK;
          mbar_expect_tx(&full[stage], CF::STAGE_BYTES);
          if constexpr (A_MN) {
#pragma unroll
            for (int j = 0; j < TM / 64; ++j)
              tma_load_2d(sa + j * (BK * 128), &map_a, &full[stage], ag0 + m0 + j * 64, ag1 + k);
          } else {
            tma_load_2d(sa, &map_a, &full[stage], ag0 + k, ag1 + m0);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * (BK * 128), &map_b, &full[stage], bg0 + n0 + j * 64, bg1 + k);
          } else {
            tma_load_2d(sb, &map_b, &full[stage], bg0 + k, bg1 + n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int g, s, m0, n0, kb0, kbn;
      decode(tile, g, s, m0, n0, kb0, kbn);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      fence_after();
      const uint32_t tmem_d = tmem_base + acc * CF::ACC_COLS;
      for (int kb = 0; kb < kbn; ++kb) {
        mbar_wait(&full[stage], phase);
        fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(smem + stage * CF::STAGE_BYTES);
          const uint32_t b_addr = a_addr + CF::A_BYTES_T;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t bd = operand_desc<B_MN>(b_addr, k);
#pragma unroll
            for (int ms = 0; ms < MS; ++ms)  // 128-row sub-tile ms: +16 KB in either major
              umma_bf16(tmem_d + ms * BN, operand_desc<A_MN>(a_addr + ms * A_BYTES, k), bd, idesc,
                        (kb | k) != 0);
          }
          umma_commit(&empty[stage]);  // smem stage free once these MMAs retire
          if (kb == kbn - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (kbn == 0 && lane == 0) umma_commit(&tfull[acc]);  // empty K range
      __syncwarp();
      if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
    uint8_t* stg = epi + ew * (2 * 32 * 128);
    int buf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int g, s, m0, n0, kb0, kbn;
      decode(tile, g, s, m0, n0, kb0, kbn);
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
#pragma unroll 1
      for (int ms = 0; ms < MS; ++ms) {
        const int row0 = m0 + ms * BM + ew * 32;  // this warp's 32 rows
        const int row = row0 + lane;
        const uint32_t tbase = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * CF::ACC_COLS + ms * BN;
        if (args.tma_epi) {
          // TMEM -> regs -> 128B-swizzled smem (32 rows x 128 B) -> TMA bulk store
          const bool rows_ok = row0 < args.M;  // M % 32 == 0 on this path
          const int64_t crow = args.c_row0 + g * args.c_grow + s * args.c_srow + row0;
          const int step = args.out_f32 ? 32 : 64;
#pragma unroll 1
          for (int c = 0; c < BN; c += step) {
            uint32_t r[64];
            tmem_ld32(tbase + c, *reinterpret_cast<uint32_t(*)[32]>(r));
            if (!args.out_f32) tmem_ld32(tbase + c + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            if (kbn == 0) {
#pragma unroll
              for (int q = 0; q < 64; ++q) r[q] = 0u;
            }
            if (args.alpha != 1.0f) {
#pragma unroll
              for (int q = 0; q < 64; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * args.alpha);
            }
            if (lane == 0) bulk_wait_read<1>();  // staging buffer `buf` free again
            __syncwarp();
            uint8_t* rowp = stg + buf * (32 * 128) + lane * 128;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              uint4 v;
              if (args.out_f32) {
                v = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
              } else {
                v.x = pack_bf16(r[8 * q + 0], r[8 * q + 1]);
                v.y = pack_bf16(r[8 * q + 2], r[8 * q + 3]);
                v.z = pack_bf16(r[8 * q + 4], r[8 * q + 5]);
                v.w = pack_bf16(r[8 * q + 6], r[8 * q + 7]);
              }
              *reinterpret_cast<uint4*>(rowp + ((q ^ (lane & 7)) * 16)) = v;
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0 && rows_ok && n0 + c < args.N) {
              if (args.accumulate)
                tma_reduce_add_2d(&map_c, stg + buf * (32 * 128), n0 + c, static_cast<int>(crow));
              else
                tma_store_2d(&map_c, stg + buf * (32 * 128), n0 + c, static_cast<int>(crow));
            }
            if (lane == 0) bulk_commit();
            buf ^= 1;
          }
          continue;
        }
        const int64_t base = g * args.c_goff + s * args.c_soff + static_cast<int64_t>(row) * args.ldc;
        const bool row_ok = row < args.M;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tbase + c, r);
          if (kbn == 0) {
#pragma unroll
            for (int q = 0; q < 32; ++q) r[q] = 0u;
          }
          if (args.alpha != 1.0f) {
#pragma unroll
            for (int q = 0; q < 32; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * args.alpha);
          }
          if (row_ok && n0 + c < args.N) {
            if (args.out_f32) {
              float4* dst = reinterpret_cast<float4*>(static_cast<float*>(args.C) + base + n0 + c);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                       __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                if (args.accumulate) {
                  const float4 o = dst[q];
                  v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                }
                dst[q] = v;
              }
            } else {
              uint4* dst =
                  reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.C) + base + n0 + c);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint4 v;
                v.x = pack_bf16(r[8 * q + 0], r[8 * q + 1]);
                v.y = pack_bf16(r[8 * q + 2], r[8 * q + 3]);
                v.z = pack_bf16(r[8 * q + 4], r[8 * q + 5]);
                v.w = pack_bf16(r[8 * q + 6], r[8 * q + 7]);
                dst[q] = v;
              }
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();  // bulk stores finished reading smem (and landed)
  }

  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(CF::TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------- CTA-pair kernel --
// 2-SM variant for the big single-group products (mm2 / adjoint): a cluster
// of two CTAs on one TPC computes a 256 x 256 tile with tcgen05.mma
// cta_group::2 (M = 256, N = 256, issued by the even CTA).  Each CTA stages
// its own 128-row half of A and 128-column half of B per K block, so per-SM
// operand traffic (smem fill and L2 reads) per FLOP halves against the
// 128 x 256 single-CTA tile; each CTA's TMEM holds its 128 rows of the
// accumulator (double-buffered, 2 x 256 columns).
//   leader  warp 0: TMA (own halves; completion to the leader's full barrier)
//           warp 1: MMA issue, commits multicast to both CTAs' barriers
//   both    warps 4..7: epilogue of their own 128 rows, TMA bulk stores;
//           release the accumulator on the leader's tempty barrier.
namespace pair {

constexpr int HALF = 128;                       // rows of A / columns of B per CTA and sub-tile
constexpr int A_B = HALF * BK * 2;              // 16 KB per 128-row A sub-tile
constexpr int B_B = HALF * BK * 2;              // 16 KB
constexpr int EPI = 4 * 2 * 32 * 128;
#ifndef POETX_PAIR_STAGES
#define POETX_PAIR_STAGES 8
#endif
// MS = 128-row A sub-tiles per CTA.  MS = 1: 256 x 256 per pair, TMEM
// accumulators double-buffered (2 x 256 columns), 6-stage ring.  MS = 2:
// 512 x 256 per pair (each CTA 256 x 256): the B stage serves two M = 256
// products, so each pair moves 48 KB per 64-deep K block for twice the
// FLOPs (0.75x the L2 -> SM bytes per FLOP; the MS = 1 kernel runs at the
// chip's L2 -> SM throughput cap on the mm2 shapes, ncu
// profiles/r02/ncu_gemm_vs_cublas.txt); the two accumulators fill TMEM, so
// the next tile starts its first stages on sub-tile 0 while the epilogue
// still drains sub-tile 1.
// Q8: B arrives as int8 codes (POET-XQ).  Warp 3 streams the codes (8 KB
// per CTA and K block, unswizzled) and their fp32 row scales into a raw
// ring that runs up to RAW_STAGES blocks ahead of the bf16 operand ring;
// converter warps (2 and 8..11) turn a raw block into the bf16 SW128 B
// operand of a free stage (code * row scale, ONE bf16 rounding: bit-identical
// to the standalone dequantizer) and arrive on the leader's full barrier.
constexpr int RAW_B = HALF * BK;                // 8 KB of int8 per CTA and K block
constexpr int RAW_S = HALF * 4;                 // + the block's row scales (<= 128 fp32)
constexpr int RAW_SLOT = RAW_B + RAW_S;
template <int MS, bool Q8 = false>
struct PCfg {
  static constexpr int STAGE = MS * A_B + B_B;
  static constexpr int FIT = (227 * 1024 - EPI - 2048) / STAGE;
  static constexpr int NQ = FIT > POETX_PAIR_STAGES ? POETX_PAIR_STAGES : FIT;   // 6 (MS 1), 4 (MS 2)
  static constexpr int STAGES = Q8 ? (MS == 1 ? 5 : 3) : NQ;
  static constexpr int RAW_FIT = (227 * 1024 - EPI - 2048 - STAGES * STAGE) / RAW_SLOT;
  static constexpr int RAW_STAGES = Q8 ? (RAW_FIT > 8 ? 8 : RAW_FIT) : 0;       // 3 (MS 1), 5 (MS 2)
  static constexpr int SMEM = STAGES * STAGE + RAW_STAGES * RAW_SLOT + EPI + 1024 + 256;
  static constexpr int TILE_M = 256 * MS;
};
// POETX_Q8_ARRIVE=cluster: converters publish with a cluster-scope release (A/B)
__device__ __forceinline__ bool q8_cta_arrive() {
#ifdef POETX_Q8_CLUSTER_ARRIVE
  return false;
#else
  return true;
#endif
}
// Q8 CTAs carry POETX_Q8_EXTRA_WARPS more warps (8..): warp 3 loads codes, warps 2 and 8.. convert
#ifndef POETX_Q8_EXTRA_WARPS
#define POETX_Q8_EXTRA_WARPS 8  /* 9 converter warps: the conversion keeps up with the MMAs (tools/q8bench.py) */
#endif
constexpr int Q8_THREADS = THREADS + 32 * POETX_Q8_EXTRA_WARPS, Q8_CONV_WARPS = 1 + POETX_Q8_EXTRA_WARPS;
// build-time timeline probe (-DPOETX_GEMM_TRACE, tools/gemmtrace.py): globaltimer
// stamps per CTA -- entry, setup done, end, and per tile: first / last MMA
// stage, epilogue start / end, first TMA issue
#ifdef POETX_GEMM_TRACE
__device__ unsigned long long g_gtrace[512 * 64];
__device__ __forceinline__ void gtr(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (slot < 64) g_gtrace[blockIdx.x * 64 + slot] = t;
}
#define GTR(slot) gtr(slot)
#else
#define GTR(slot) ((void)(slot))
#endif
// 512-row tiles: K blocks at the end of a tile that run sub-tile 0 first
// (0: both sub-tiles interleaved to the end, as round 2 first shipped)
#ifndef POETX_PAIR_TAIL
#define POETX_PAIR_TAIL 3
#endif
// timeline probe knob (-DPOETX_EPI_PROBE=1: no TMA stores); results invalid
#ifndef POETX_EPI_PROBE
#define POETX_EPI_PROBE 0
#endif
template <int MS, bool A_MN, bool B_MN, bool Q8 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Q8 ? Q8_THREADS : THREADS, 1)
    tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_c, Args args) {
  using PC = PCfg<MS, Q8>;
  constexpr int STAGES = PC::STAGES, STAGE = PC::STAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = /* 1024-byte aligned, kept in the shared address space (STS/LDS) */ smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi = smem + STAGES * STAGE;
  constexpr int RSTG = PC::RAW_STAGES;
  uint8_t* rawring = epi + EPI;  // Q8 only: RSTG x (codes + scales)
  uint64_t* full = reinterpret_cast<uint64_t*>(rawring + RSTG * RAW_SLOT);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rawfull = tempty + 2;  // Q8 only: RSTG each
  uint64_t* rawempty = rawfull + RSTG;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rawempty + RSTG);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int tiles_per_split = args.m_tiles * args.n_tiles;  // TILE_M x 256 tiles
  const int num_tiles = tiles_per_split * args.splits * args.groups;

  // tile -> group, K split, row / 256-column origin, K-block range
  auto decode = [&](int tile, int& g, int& s, int& m0, int& n0, int& kb0, int& kbn) {
    g = tile / (tiles_per_split * args.splits);
    int r = tile % (tiles_per_split * args.splits);
    s = r / tiles_per_split;
    r %= tiles_per_split;
    m0 = (r / args.n_tiles) * PC::TILE_M;
    n0 = (r % args.n_tiles) * 256;
    const int k0 = s * args.kps;
    const int k1 = k0 + args.kps < args.K ? k0 + args.kps : args.K;
    kb0 = k0 / BK;
    kbn = (k1 - k0 + BK - 1) / BK;
  };

  if (threadIdx.x == 0) {
    GTR(0);
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], Q8 ? 3 : 1);  // Q8: + one elected converter thread in each CTA
      mbar_init(&empty[st], 1);
    }
    for (int st = 0; st < RSTG; ++st) {
      mbar_init(&rawfull[st], 1);
      mbar_init(&rawempty[st], Q8_CONV_WARPS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps in each CTA of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GTR(1);

  if (Q8 && warp == 3) {
    // codes + row scales of every K block of this CTA's B half, RSTG blocks ahead
    if (lane == 0) {
      int rs = 0;
      uint32_t rph = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        int g, sp, m0, n0, kb0, kbn;
        decode(tile, g, sp, m0, n0, kb0, kbn);
        const int bn = n0 + rank * HALF;
        const int bg0 = args.b_g0 * g, bg1 = args.b_g1 * g;
        for (int kb = kb0; kb < kb0 + kbn; ++kb) {
          mbar_wait(&rawempty[rs], rph ^ 1);
          uint8_t* raw = rawring + rs * RAW_SLOT;
          const int k = kb * BK;
          const int srow = B_MN ? bg1 + k : bg1 + bn;  // first B row of the block
          const int nsc = B_MN ? BK : HALF;
          mbar_expect_tx(&rawfull[rs], RAW_B + nsc * 4);
          if constexpr (B_MN)
            tma_load_2d(raw, &map_b, &rawfull[rs], bg0 + bn, bg1 + k);
          else
            tma_load_2d(raw, &map_b, &rawfull[rs], bg0 + k, bg1 + bn);
          bulk_load_1d(raw + RAW_B, args.bscale + srow, nsc * 4, &rawfull[rs]);
          if (++rs == RSTG) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (Q8 && (warp == 2 || warp >= 8)) {
    // int8 -> bf16 B converter: this CTA's half (128 B columns) of every stage
    const int ct = (warp == 2 ? 0 : warp - 7) * 32 + lane;  // 0 .. 32 * Q8_CONV_WARPS - 1
    int stage = 0, rs = 0;
    uint32_t phase = 0, rph = 0;
    for (int tile = cluster; tile < num_tiles; tile += nclusters) {
      int g, sp, m0, n0, kb0, kbn;
      decode(tile, g, sp, m0, n0, kb0, kbn);
      for (int kb = kb0; kb < kb0 + kbn; ++kb) {
        mbar_wait(&rawfull[rs], rph);
        mbar_wait(&empty[stage], phase ^ 1);  // the bf16 stage is free (MMAs done with it)
        const uint8_t* raw = rawring + rs * RAW_SLOT;
        const float* scl = reinterpret_cast<const float*>(raw + RAW_B);
        uint8_t* sb = smem + stage * STAGE + MS * A_B;
#pragma unroll 2
        for (int u = ct; u < HALF * BK / 8; u += 32 * Q8_CONV_WARPS) {
          int r, c;  // raw row / first of 8 columns (raw rows are 128 B (MN) or 64 B (K-major))
          uint32_t dst;
          if constexpr (B_MN) {  // raw [64 K rows][128 N cols], scale per K row
            r = u >> 4;
            c = (u & 15) * 8;
            dst = static_cast<uint32_t>((c >> 6) * (BK * 128) + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4));
          } else {               // raw [128 N rows][64 K cols], scale per N row
            r = u >> 3;
            c = (u & 7) * 8;
            dst = static_cast<uint32_t>(r * 128 + (((c >> 3) ^ (r & 7)) << 4));
          }
          const float sc = scl[r];
          const uint2 q = *reinterpret_cast<const uint2*>(raw + r * (B_MN ? HALF : BK) + c);
          // int8 -> fp32 without I2F: byte b (biased by +128) into the mantissa
          // of 2^23 (PRMT), minus 2^23 + 128 (exact); then code * scale and ONE
          // bf16 rounding, as the standalone dequantizer
          const uint32_t w[2] = {q.x ^ 0x80808080u, q.y ^ 0x80808080u};
          uint32_t h[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const uint32_t src = w[x >> 1], sel0 = 0x7540u | ((x & 1) * 2), sel1 = 0x7541u | ((x & 1) * 2);
            const float f0 = (__uint_as_float(__byte_perm(src, 0x4B000000u, sel0)) - 8388736.0f) * sc;
            const float f1 = (__uint_as_float(__byte_perm(src, 0x4B000000u, sel1)) - 8388736.0f) * sc;
            __nv_bfloat162 v = __floats2bfloat162_rn(f0, f1);
            h[x] = *reinterpret_cast<uint32_t*>(&v);
          }
          *reinterpret_cast<uint4*>(sb + dst) = make_uint4(h[0], h[1], h[2], h[3]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&rawempty[rs]);
        // every converter warp's stores are in (named barrier 1 over the
        // converter warps), then ONE cluster-scope release arrival per CTA
        asm volatile("bar.sync 1, %0;" ::"n"(32 * Q8_CONV_WARPS) : "memory");
        if (ct == 0) {
          if (q8_cta_arrive()) arrive_leader_cta(&full[stage]);
          else arrive_leader(&full[stage]);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (++rs == RSTG) { rs = 0; rph ^= 1; }
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        int g, sp, m0, n0, kb0, kbn;
        decode(tile, g, sp, m0, n0, kb0, kbn);
        const int bn = n0 + rank * HALF;  // this CTA's half of B
        const int ag0 = args.a_g0 * g, ag1 = args.a_g1 * g, bg0 = args.b_g0 * g, bg1 = args.b_g1 * g;
        const int tj = (tile - cluster) / nclusters;
        for (int kb = kb0; kb < kb0 + kbn; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (kb == kb0) GTR(4 + tj * 5 + 4);
          uint8_t* sa = smem + stage * STAGE;
          uint8_t* sb = sa + MS * A_B;
          const uint32_t fb = smem_u32(&full[stage]) & PEER_MASK;
          if (leader) mbar_expect_tx(&full[stage], 2 * (Q8 ? MS * A_B : STAGE));
          const int k = kb * BK;
#pragma unroll
          for (int h = 0; h < MS; ++h) {
            const int am = m0 + h * 256 + rank * HALF;  // this CTA's rows of sub-tile h
            if constexpr (A_MN) {
#pragma unroll
              for (int j = 0; j < HALF / 64; ++j)
                tma_load_2sm(sa + h * A_B + j * (BK * 128), &map_a, fb, ag0 + am + j * 64, ag1 + k);
            } else {
              tma_load_2sm(sa + h * A_B, &map_a, fb, ag0 + k, ag1 + am);
            }
          }
          if constexpr (Q8) {
            // B: the converter warps fill it from the raw ring (warp 3 loads the codes)
          } else if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < HALF / 64; ++j) tma_load_2sm(sb + j * (BK * 128), &map_b, fb, bg0 + bn + j * 64, bg1 + k);
          } else {
            tma_load_2sm(sb, &map_b, fb, bg0 + k, bg1 + bn);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16(256, 256, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      // one 256 x 256 x 64 product set from a stage's A sub-tile h into TMEM column d
      auto mma_stage = [&](int st, int h, uint32_t d, bool acc) {
        const uint32_t a_addr = smem_u32(smem + st * STAGE) + h * A_B;
        const uint32_t b_addr = smem_u32(smem + st * STAGE) + MS * A_B;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma2_bf16(d, operand_desc<A_MN>(a_addr, k), operand_desc<B_MN>(b_addr, k), idesc, (acc || k) ? 1u : 0u);
      };
      if constexpr (MS == 1) {
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = cluster; tile < num_tiles; tile += nclusters) {
          int g, sp, m0, n0, kb0, kbn;
          decode(tile, g, sp, m0, n0, kb0, kbn);
          wait_cluster(&tempty[acc], acc_phase ^ 1);
          fence_after();
          const uint32_t tmem_d = tmem_base + acc * 256;
          const int tj = (tile - cluster) / nclusters;
          for (int kb = 0; kb < kbn; ++kb) {
            mbar_wait(&full[stage], phase);
            fence_after();
            if (lane == 0) {
              if (kb == 0) GTR(4 + tj * 5 + 0);
              mma_stage(stage, 0, tmem_d, kb != 0);
              commit2(&empty[stage]);
              if (kb == kbn - 1) { commit2(&tfull[acc]); GTR(4 + tj * 5 + 1); }
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (kbn == 0 && lane == 0) commit2(&tfull[acc]);  // empty K range
          __syncwarp();
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      } else {
        uint32_t tph = 0;
        for (int tile = cluster; tile < num_tiles; tile += nclusters) {
          int g, sp, m0, n0, kb0, kbn;
          decode(tile, g, sp, m0, n0, kb0, kbn);
          const int lead = kbn < STAGES ? kbn : STAGES;
          // the last `tail` K blocks run sub-tile 0 first (stages held), so its
          // accumulator completes -- and the epilogue starts draining it --
          // while sub-tile 1 finishes: the next tile's first MMA waits for
          // that drain (single-buffered TMEM), now mostly hidden
          const int tail = kbn > lead ? (POETX_PAIR_TAIL < kbn - lead ? POETX_PAIR_TAIL : kbn - lead) : 0;
          const int tj = (tile - cluster) / nclusters;
          // sub-tile 0 starts on the first `lead` stages as soon as its
          // accumulator is drained; sub-tile 1 follows on the same (held)
          // stages once the epilogue has drained its accumulator too
          wait_cluster(&tempty[0], tph ^ 1);
          fence_after();
          const int st0 = stage;
          const uint32_t ph0 = phase;
          for (int kb = 0; kb < lead; ++kb) {
            mbar_wait(&full[stage], phase);
            fence_after();
            if (kb == 0 && lane == 0) GTR(4 + tj * 5 + 0);
            if (lane == 0) {
              mma_stage(stage, 0, tmem_base, kb != 0);
              if (kb == kbn - 1) commit2(&tfull[0]);
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          wait_cluster(&tempty[1], tph ^ 1);
          fence_after();
          stage = st0;
          phase = ph0;
          for (int kb = 0; kb < lead; ++kb) {
            if (lane == 0) {
              mma_stage(stage, 1, tmem_base + 256, kb != 0);
              commit2(&empty[stage]);
              if (kb == kbn - 1) commit2(&tfull[1]);
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          for (int kb = lead; kb < kbn - tail; ++kb) {
            mbar_wait(&full[stage], phase);
            fence_after();
            if (lane == 0) {
              mma_stage(stage, 0, tmem_base, true);
              mma_stage(stage, 1, tmem_base + 256, true);
              commit2(&empty[stage]);
              if (kb == kbn - 1) {  // no tail
                commit2(&tfull[0]);
                commit2(&tfull[1]);
                GTR(4 + tj * 5 + 1);
              }
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          if (tail > 0) {
            const int st1 = stage;
            const uint32_t ph1 = phase;
            for (int kb = kbn - tail; kb < kbn; ++kb) {
              mbar_wait(&full[stage], phase);
              fence_after();
              if (lane == 0) {
                mma_stage(stage, 0, tmem_base, true);
                if (kb == kbn - 1) commit2(&tfull[0]);
              }
              __syncwarp();
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            stage = st1;
            phase = ph1;
            for (int kb = kbn - tail; kb < kbn; ++kb) {
              if (lane == 0) {
                mma_stage(stage, 1, tmem_base + 256, true);
                commit2(&empty[stage]);
                if (kb == kbn - 1) { commit2(&tfull[1]); GTR(4 + tj * 5 + 1); }
              }
              __syncwarp();
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          }
          if (kbn == 0 && lane == 0) {  // empty K range
            commit2(&tfull[0]);
            commit2(&tfull[1]);
          }
          __syncwarp();
          tph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    uint8_t* stg = epi + ew * (2 * 32 * 128);
    int buf = 0, acc = 0;
    uint32_t acc_phase = 0;
    const int step = args.out_f32 ? 32 : 64;
    for (int tile = cluster; tile < num_tiles; tile += nclusters) {
      int g, sp, m0, n0, kb0, kbn;
      decode(tile, g, sp, m0, n0, kb0, kbn);
      // MS = 1: one accumulator per tile; MS = 2: sub-tile h completes on tfull[h]
      mbar_wait(&tfull[MS == 1 ? acc : 0], acc_phase);
      fence_after();
      const int tj = (tile - cluster) / nclusters;
      if (ew == 0 && lane == 0) GTR(4 + tj * 5 + 2);
#pragma unroll 1
      for (int h = 0; h < MS; ++h) {
        if (MS == 2 && h == 1) {
          mbar_wait(&tfull[1], acc_phase);
          fence_after();
        }
        const int row0 = m0 + h * 256 + rank * HALF + ew * 32;  // this warp's 32 rows (within the group)
        const int64_t crow = args.c_row0 + g * args.c_grow + sp * args.c_srow + row0;
        const uint32_t tbase = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + (MS == 1 ? acc : h) * 256;
#pragma unroll 1
        for (int c = 0; c < 256; c += step) {
          uint32_t r[64];
          tmem_ld32(tbase + c, *reinterpret_cast<uint32_t(*)[32]>(r));
          if (!args.out_f32) tmem_ld32(tbase + c + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
          if (kbn == 0) {
#pragma unroll
            for (int q = 0; q < 64; ++q) r[q] = 0u;
          }
          if (args.alpha != 1.0f) {
#pragma unroll
            for (int q = 0; q < 64; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * args.alpha);
          }
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          uint8_t* rowp = stg + buf * (32 * 128) + lane * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4 v;
            if (args.out_f32) {
              v = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
            } else {
              v.x = pack_bf16(r[8 * q + 0], r[8 * q + 1]);
              v.y = pack_bf16(r[8 * q + 2], r[8 * q + 3]);
              v.z = pack_bf16(r[8 * q + 4], r[8 * q + 5]);
              v.w = pack_bf16(r[8 * q + 6], r[8 * q + 7]);
            }
            *reinterpret_cast<uint4*>(rowp + ((q ^ (lane & 7)) * 16)) = v;
          }
          fence_async_smem();
          __syncwarp();
          if (POETX_EPI_PROBE != 1 && lane == 0 && row0 < args.M && n0 + c < args.N) {
            if (args.accumulate)
              tma_reduce_add_2d(&map_c, stg + buf * (32 * 128), n0 + c, static_cast<int>(crow));
            else
              tma_store_2d(&map_c, stg + buf * (32 * 128), n0 + c, static_cast<int>(crow));
          }
          if (lane == 0) bulk_commit();
          buf ^= 1;
        }
        fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[MS == 1 ? acc : h]);
        if (tj == 0 && ew == 0 && lane == 0) GTR(60 + h);
      }
      if (ew == 0 && lane == 0) GTR(4 + tj * 5 + 3);
      if (MS == 1) {
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      } else {
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  fence_before();
  cluster_sync();
  fence_after();
  if (threadIdx.x == 0) GTR(2);
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

}  // namespace pair

// -------------------------------------------------------------- host side --
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// cuTensorMapEncodeTiled is a driver call: make sure the calling thread has
// the device's primary context current (autograd's backward worker threads
// may not have touched the runtime yet; tools such as ncu / compute-sanitizer
// then reject the encode with CUDA_ERROR_INVALID_CONTEXT)
static void ensure_context() {
  thread_local bool done = false;
  if (!done) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaSetDevice(dev);
    done = true;
  }
}

// 2-D bf16 tensor map over a row-major [rows, cols] view with row pitch
int make_map(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
             uint32_t box_cols, uint32_t box_rows) {
  ensure_context();
  auto fn = encode_fn();
  POETX_REQUIRE(fn != nullptr, POETX_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  POETX_REQUIRE(r == CUDA_SUCCESS, POETX_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return POETX_OK;
}

int make_map_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
                 uint32_t box_cols, uint32_t box_rows) {
  ensure_context();
  auto fn = encode_fn();
  POETX_REQUIRE(fn != nullptr, POETX_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  POETX_REQUIRE(r == CUDA_SUCCESS, POETX_ECUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", (int)r);
  return POETX_OK;
}

// 2-D int8 tensor map (unswizzled) over a row-major [rows, cols] view, pitch in bytes
int make_map_u8(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
                uint32_t box_cols, uint32_t box_rows) {
  ensure_context();
  auto fn = encode_fn();
  POETX_REQUIRE(fn != nullptr, POETX_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  POETX_REQUIRE(r == CUDA_SUCCESS, POETX_ECUDA, "cuTensorMapEncodeTiled (u8) failed (%d)", (int)r);
  return POETX_OK;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN, int MS>
int launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const Args& a,
             const char* name, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc_kernel<BN, A_MN, B_MN, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg<BN, MS>::SMEM_BYTES);
    attr_set = true;
  }
  int64_t tiles = static_cast<int64_t>(a.m_tiles) * a.n_tiles * a.splits * a.groups;
  int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
  if (grid <= 0) return POETX_OK;
  void* tok = prof_begin(st);
  tc_kernel<BN, A_MN, B_MN, MS><<<grid, THREADS, Cfg<BN, MS>::SMEM_BYTES, st>>>(ma, mb, mc, a);
  prof_end(tok, name, 2.0 * a.M * a.N * static_cast<double>(a.K) * a.groups, st);
  POETX_LAUNCHED(name);
  return POETX_OK;
}

template <int BN>
int launch_bn(bool a_mn, bool b_mn, int ms, const CUtensorMap& ma, const CUtensorMap& mb,
              const CUtensorMap& mc, const Args& a, const char* name, cudaStream_t st) {
  if (ms == 2) {
    if (a_mn && b_mn) return launch_t<BN, true, true, 2>(ma, mb, mc, a, name, st);
    return POETX_ENOTSUPPORTED;
  }
  if (!a_mn && !b_mn) return launch_t<BN, false, false, 1>(ma, mb, mc, a, name, st);
  if (!a_mn && b_mn) return launch_t<BN, false, true, 1>(ma, mb, mc, a, name, st);
  if (a_mn && !b_mn) return launch_t<BN, true, false, 1>(ma, mb, mc, a, name, st);
  return launch_t<BN, true, true, 1>(ma, mb, mc, a, name, st);
}

}  // namespace tc

static int g_pair_on = [] {
  const char* e = getenv("POETX_GEMM_PAIR");
  return e && e[0] == '0' ? 0 : 1;
}();
// A sub-tiles per pair CTA: 0 = by shape, 1 / 2 forced (POETX_PAIR_MS, A/B)
static int g_pair_ms = [] {
  const char* e = getenv("POETX_PAIR_MS");
  return e ? atoi(e) : 0;
}();
// 512 x 256 pair tiles for one single-split product with M >= 512 (mm2 /
// adjoint); grouped and split-K products keep 256 x 256
static int pair_ms(const TcProblem& p, int nblk, bool q8 = false) {
  if (nblk != 1 || p.M < 512) return 1;
  (void)q8;  // int8 B: 512-row tiles too (half the conversions per FLOP; tools/q8bench.py)
  if (g_pair_ms == 1 || g_pair_ms == 2) return g_pair_ms;
  // whole tile rounds on the SM pairs, a 512-row tile costing two 256-row
  // ones less the ~5% its halved L2 -> SM traffic buys: e.g. 8192 x 2816
  // (352 vs 176 tiles on 74 pairs: 5 rounds vs 3 x 1.9) keeps 256 rows,
  // 8192 x 5632 (10 vs 5 x 1.9) and 8192 x 2048 (4 vs 2 x 1.9) take 512
  const int64_t pairs = tc::num_sms() / 2, nt = p.N / 256;
  const int64_t r1 = ((p.M + 255) / 256 * nt + pairs - 1) / pairs;
  const int64_t r2 = ((p.M + 511) / 512 * nt + pairs - 1) / pairs;
  return 1.9 * r2 < r1 ? 2 : 1;
}

namespace tc {
template <int MS, bool A_MN, bool B_MN, bool Q8 = false>
int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const Args& a,
                const char* name, cudaStream_t st) {
  using PC = pair::PCfg<MS, Q8>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(pair::tc2_kernel<MS, A_MN, B_MN, Q8>, cudaFuncAttributeMaxDynamicSharedMemorySize, PC::SMEM);
    attr_set = true;
  }
  const int64_t tiles = static_cast<int64_t>(a.m_tiles) * a.n_tiles * a.splits * a.groups;
  const int64_t pairs = num_sms() / 2;
  const int grid = static_cast<int>(2 * (tiles < pairs ? tiles : pairs));
  if (grid <= 0) return POETX_OK;
  void* tok = prof_begin(st);
  pair::tc2_kernel<MS, A_MN, B_MN, Q8><<<grid, Q8 ? pair::Q8_THREADS : THREADS, PC::SMEM, st>>>(ma, mb, mc, a);
  prof_end(tok, name, 2.0 * a.M * a.N * static_cast<double>(a.K) * a.groups, st);
  POETX_LAUNCHED(name);
  return POETX_OK;
}
template <int MS, bool Q8>
int launch_pair_ms(bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                   const Args& a, const char* name, cudaStream_t st) {
  if (a_mn)
    return b_mn ? launch_pair<MS, true, true, Q8>(ma, mb, mc, a, name, st)
                : launch_pair<MS, true, false, Q8>(ma, mb, mc, a, name, st);
  return b_mn ? launch_pair<MS, false, true, Q8>(ma, mb, mc, a, name, st)
              : launch_pair<MS, false, false, Q8>(ma, mb, mc, a, name, st);
}
}  // namespace tc

// An operand is a row-major [rows, cols] bf16 view with a row pitch.
// K-major: the contraction index runs along cols; MN-major: along rows.
int tc_grouped(const TcOperand& A, const TcOperand& B, const TcProblem& p, cudaStream_t st) {
  using namespace tc;
  const int BN = p.bn;
  POETX_REQUIRE(BN == 64 || BN == 128 || BN == 256, POETX_ESHAPE, "tc: bad BN %d", BN);
  if (p.M <= 0 || p.N <= 0 || p.groups <= 0) return POETX_OK;
  const bool q8 = B.row_scale != nullptr;
  if (A.row_scale) return POETX_ENOTSUPPORTED;
  for (const TcOperand* o : {&A, &B}) {
    if ((reinterpret_cast<uintptr_t>(o->ptr) & 15) || (o->pitch % (o == &B && q8 ? 16 : 8))) return POETX_ENOTSUPPORTED;
  }
  if ((reinterpret_cast<uintptr_t>(p.C) & 15) || (p.ldc % 8) || (p.c_goff % 8) || (p.c_soff % 8))
    return POETX_ENOTSUPPORTED;
  if (p.N % 32) return POETX_ENOTSUPPORTED;
  // CTA pair: 256 x 256 tiles; N whole tiles (groups may sit side by side in C),
  // M whole tiles unless a single (group, split) block owns all rows of C
  const int nblk = p.groups * (p.splits < 1 ? 1 : p.splits);
  if (g_pair_on && p.ms != 2 && p.N % 256 == 0 && (p.M % 256 == 0 || nblk == 1) && p.tma_epi &&
      p.c_goff % p.ldc == 0 && p.c_soff % p.ldc == 0 && (p.ldc * (p.out_f32 ? 4 : 2)) % 16 == 0 &&
      !(p.accumulate && !p.out_f32)) {
    CUtensorMap pa, pb, pc;
    POETX_TRY(make_map(&pa, A.ptr, A.cols, A.rows, A.pitch, 64, A.mn_major ? BK : pair::HALF));
    if (q8)  // int8 codes, unswizzled raw boxes: {128 N, 64 K} (MN-major) or {64 K, 128 N}
      POETX_TRY(make_map_u8(&pb, B.ptr, B.cols, B.rows, B.pitch, B.mn_major ? pair::HALF : BK,
                            B.mn_major ? BK : pair::HALF));
    else
      POETX_TRY(make_map(&pb, B.ptr, B.cols, B.rows, B.pitch, 64, B.mn_major ? BK : pair::HALF));
    Args a{};
    a.M = static_cast<int>(p.M);
    a.N = static_cast<int>(p.N);
    a.K = static_cast<int>(p.K);
    a.groups = p.groups;
    a.splits = p.splits < 1 ? 1 : p.splits;
    int64_t kps = (p.K + a.splits - 1) / a.splits;
    kps = (kps + BK - 1) / BK * BK;
    a.kps = static_cast<int>(kps > 0 ? kps : BK);
    // 512-row pair tiles for single products tall enough to use them
    const int ms = pair_ms(p, nblk, q8);
    a.m_tiles = static_cast<int>((p.M + 256 * ms - 1) / (256 * ms));
    a.n_tiles = static_cast<int>(p.N / 256);
    a.a_g0 = p.a_g0; a.a_g1 = p.a_g1; a.b_g0 = p.b_g0; a.b_g1 = p.b_g1;
    a.C = p.C;
    a.ldc = p.ldc; a.c_goff = p.c_goff; a.c_soff = p.c_soff;
    a.out_f32 = p.out_f32;
    a.accumulate = p.accumulate;
    a.alpha = p.alpha;
    a.tma_epi = 1;
    a.c_row0 = 0;
    a.c_grow = p.c_goff / p.ldc;
    a.c_srow = p.c_soff / p.ldc;
    a.bscale = B.row_scale;
    const int64_t rows = (p.groups - 1) * a.c_grow + (a.splits - 1) * a.c_srow + p.M;
    POETX_TRY(p.out_f32 ? make_map_f32(&pc, p.C, p.N, rows, p.ldc, 32, 32) : make_map(&pc, p.C, p.N, rows, p.ldc, 64, 32));
    const char* nm = p.name ? p.name : "tc_gemm";
    if (q8)
      return ms == 2 ? launch_pair_ms<2, true>(A.mn_major, B.mn_major, pa, pb, pc, a, nm, st)
                     : launch_pair_ms<1, true>(A.mn_major, B.mn_major, pa, pb, pc, a, nm, st);
    return ms == 2 ? launch_pair_ms<2, false>(A.mn_major, B.mn_major, pa, pb, pc, a, nm, st)
                   : launch_pair_ms<1, false>(A.mn_major, B.mn_major, pa, pb, pc, a, nm, st);
  }
  if (q8) return POETX_ENOTSUPPORTED;  // int8 B: pair kernel only
  CUtensorMap ma, mb;
  const int ms = p.ms == 2 ? 2 : 1;
  POETX_TRY(make_map(&ma, A.ptr, A.cols, A.rows, A.pitch, 64, A.mn_major ? BK : BM * ms));
  POETX_TRY(make_map(&mb, B.ptr, B.cols, B.rows, B.pitch, 64, B.mn_major ? BK : BN));
  Args a{};
  a.M = static_cast<int>(p.M);
  a.N = static_cast<int>(p.N);
  a.K = static_cast<int>(p.K);
  a.groups = p.groups;
  a.splits = p.splits < 1 ? 1 : p.splits;
  int64_t kps = (p.K + a.splits - 1) / a.splits;
  kps = (kps + BK - 1) / BK * BK;
  a.kps = static_cast<int>(kps > 0 ? kps : BK);
  a.m_tiles = static_cast<int>((p.M + BM * ms - 1) / (BM * ms));
  a.n_tiles = static_cast<int>((p.N + BN - 1) / BN);
  a.a_g0 = p.a_g0; a.a_g1 = p.a_g1; a.b_g0 = p.b_g0; a.b_g1 = p.b_g1;
  a.C = p.C;
  a.ldc = p.ldc; a.c_goff = p.c_goff; a.c_soff = p.c_soff;
  a.out_f32 = p.out_f32;
  a.accumulate = p.accumulate;
  if (p.accumulate && !p.out_f32) return POETX_ENOTSUPPORTED;
  // TMA-store epilogue when every (group, split) block of C starts on a row of
  // one 2-D view of C and rows come in whole 32-row warp chunks
  CUtensorMap mc;
  memset(&mc, 0, sizeof(mc));
  a.tma_epi = 0;
  if (p.tma_epi && p.M % 32 == 0 && p.c_goff % p.ldc == 0 && p.c_soff % p.ldc == 0 &&
      (p.ldc * (p.out_f32 ? 4 : 2)) % 16 == 0) {
    a.c_row0 = 0;
    a.c_grow = p.c_goff / p.ldc;
    a.c_srow = p.c_soff / p.ldc;
    const int64_t rows = (p.groups - 1) * a.c_grow + (a.splits - 1) * a.c_srow + p.M;
    int rc = p.out_f32 ? make_map_f32(&mc, p.C, p.N, rows, p.ldc, 32, 32)
                       : make_map(&mc, p.C, p.N, rows, p.ldc, 64, 32);
    if (rc == POETX_OK) a.tma_epi = 1;
  }
  a.alpha = p.alpha;
  const char* name = p.name ? p.name : "tc_gemm";
  if (BN == 256) return launch_bn<256>(A.mn_major, B.mn_major, ms, ma, mb, mc, a, name, st);
  if (BN == 128) return launch_bn<128>(A.mn_major, B.mn_major, ms, ma, mb, mc, a, name, st);
  return launch_bn<64>(A.mn_major, B.mn_major, ms, ma, mb, mc, a, name, st);
}

int tc_matmul(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA,
              const void* B, int64_t ldb, int transB, void* C, int64_t ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return POETX_OK;
  if (K <= 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return POETX_ENOTSUPPORTED;

  // op(A)[M,K]: stored [M,K] (K-major) or [K,M] (MN-major)
  TcOperand a{A, transA ? K : M, transA ? M : K, lda, transA != 0};
  // op(B)[K,N]: stored [K,N] (MN-major) or [N,K] (K-major)
  TcOperand b{B, transB ? N : K, transB ? K : N, ldb, transB == 0};
  TcProblem p{};
  p.M = M; p.N = N; p.K = K; p.groups = 1; p.splits = 1; p.bn = 256;
  p.C = C; p.ldc = ldc; p.alpha = 1.0f; p.name = "tc_gemm"; p.tma_epi = 1;
  return tc_grouped(a, b, p, st);
}

int tc_matmul_q8(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA, const int8_t* B,
                 int64_t ldb, int transB, const float* scales, void* C, int64_t ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return POETX_OK;
  if (K <= 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || !scales) return POETX_ENOTSUPPORTED;
  TcOperand a{A, transA ? K : M, transA ? M : K, lda, transA != 0};
  TcOperand b{B, transB ? N : K, transB ? K : N, ldb, transB == 0, scales};
  TcProblem p{};
  p.M = M; p.N = N; p.K = K; p.groups = 1; p.splits = 1; p.bn = 256;
  p.C = C; p.ldc = ldc; p.alpha = 1.0f; p.name = "tc_gemm_q8"; p.tma_epi = 1;
  return tc_grouped(a, b, p, st);
}

int tc_blockdiag(const GemmDesc& d, cudaStream_t st) {
  // apply_to_features: A = x [T, dim] K-major with group column offset b;
  // B = G stack [nb*b, b] (MN-major for G, K-major for G^T) with row offset b
  const int64_t b = d.K, nb = d.batch, dim = d.sAm, T = d.M;
  if (b % 64 || b > 256 || d.N != b || d.sAk != 1 || d.sAb != b || d.sCm != dim ||
      d.sCb != b || d.sCn != 1 || d.sBb != b * b)
    return POETX_ENOTSUPPORTED;
  const bool trans = d.sBk == 1;
  return tc_blockdiag_apply(T, nb, b, d.B, trans ? 1 : 0, d.A, d.C, st);
}

size_t tc_outer_ws_bytes(int64_t T, int64_t nb, int64_t b) {
  int s = tc_outer_splits(T, nb, b);
  return s > 1 ? align_up(static_cast<size_t>(s) * nb * b * b * 4) : 0;
}

int tc_outer_splits(int64_t T, int64_t nb, int64_t b) {
  int64_t bn = b < 256 ? b : 256;
  int64_t tm = 128;
  int64_t tiles = nb * ((b + tm - 1) / tm) * ((b + bn - 1) / bn);
  // one wave of persistent CTAs: fewer fp32 partials to write and reduce
  // SM share (percent) the split count targets.  The outer products run on a
  // side stream next to the main chain (layer.cu), so a partial share wins:
  // fewer fp32 partials to write and reduce, the rest of the SMs stay with the
  // chain (Llama-1B step: 100% -> 98.9k tok/s, 25-50% -> 101.5k)
  static const int64_t share = [] {
    const char* e = getenv("POETX_OUTER_SM_PCT");
    return static_cast<int64_t>(e ? atoi(e) : 40);
  }();
  int64_t want = (148 * share / 100) / tiles;
  int64_t maxs = (T + 511) / 512;
  if (want > maxs) want = maxs;
  if (want < 1) want = 1;
  if (want > 64) want = 64;
  return static_cast<int>(want);
}

}  // namespace poetx

extern "C" int poetx_tc_enabled(void) { return poetx::g_tc_on; }
extern "C" int poetx_gemm_pair_enabled(void) { return poetx::g_pair_on; }
extern "C" void poetx_set_gemm_pair_enabled(int on) { poetx::g_pair_on = on ? 1 : 0; }
extern "C" void poetx_set_gemm_pair_ms(int ms) { poetx::g_pair_ms = ms; }
extern "C" void poetx_set_tc_enabled(int on) { poetx::g_tc_on = on ? 1 : 0; }

#ifdef POETX_GEMM_TRACE
extern "C" int poetx_gemm_trace_copy(unsigned long long* host, int n) {
  if (n > 512 * 64) n = 512 * 64;
  return static_cast<int>(cudaMemcpyFromSymbol(host, poetx::tc::pair::g_gtrace, n * sizeof(unsigned long long)));
}
extern "C" int poetx_gemm_trace_reset() {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, poetx::tc::pair::g_gtrace) != cudaSuccess) return 1;
  return static_cast<int>(cudaMemset(p, 0, sizeof(poetx::tc::pair::g_gtrace)));
}
#endif
