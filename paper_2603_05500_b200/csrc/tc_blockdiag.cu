// Block-diagonal factor application on tensor cores (apply_to_features,
// blockdiag.py:58-73) for the BF16 path:
//
//     y[:, s*b:(s+1)*b] = x[:, s*b:(s+1)*b] . G[s]      (or G[s]^T)
//
// This op sits below the ridge point (b/2 FLOP per byte), so the kernel is
// organised around HBM traffic, not MMA issue:
//   * every CTA owns ONE block s and a contiguous range of 128-token tiles;
//     G[s] (b x b bf16, <= 128 KB) is loaded into shared memory ONCE and
//     stays resident, so G costs ~nothing next to the activation stream
//     (a plain tiled GEMM re-reads G per token tile: 2x the x traffic);
//   * the x tiles stream through a 4-stage TMA ring (SWIZZLE_128B);
//   * tcgen05.mma (M=128, N=b, K=16) accumulates in a double-buffered TMEM
//     accumulator, so tile i+1's MMAs overlap tile i's epilogue;
//   * epilogue: tcgen05.ld -> bf16 -> 128B-swizzled smem staging (per warp,
//     double-buffered) -> TMA bulk-tensor store: full-line coalesced writes.
#include <cudaTypedefs.h>

#include "tc_common.cuh"
#include "tc_gemm.cuh"

namespace poetx {

void* prof_begin(cudaStream_t st);
void prof_end(void* token, const char* name, double flops, cudaStream_t st);

namespace tc {
namespace {

constexpr int BD_THREADS = 256;
#ifndef POETX_BD_STAGES
#define POETX_BD_STAGES 4
#endif
#ifndef POETX_BD_EPI_BUFS
#define POETX_BD_EPI_BUFS 2
#endif
constexpr int BD_STAGES = POETX_BD_STAGES;
constexpr int BD_EPI_BUFS = POETX_BD_EPI_BUFS;
constexpr int BD_A_BYTES = BM * BK * 2;          // 16 KB x tile
constexpr int BD_EPI_BYTES = 4 * BD_EPI_BUFS * 32 * 128;  // 4 warps x buffers x (32 rows x 128 B)

template <int BN> struct BdCfg {
  static constexpr int B_BYTES = BN * BN * 2;  // resident G[s]
  static constexpr int SMEM = B_BYTES + BD_STAGES * BD_A_BYTES + BD_EPI_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 2 * BN;
};

struct BdArgs {
  int T, b, m_tiles, chunks, per;
};

template <int BN, bool B_MN>
__global__ void __launch_bounds__(BD_THREADS, 1)
    bd_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_g,
              const __grid_constant__ CUtensorMap map_y, BdArgs args) {
  using CF = BdCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = /* 1024-byte aligned, kept in the shared address space (STS/LDS) */ smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sg = smem;                                   // resident G[s]
  uint8_t* ring = sg + CF::B_BYTES;                     // x tiles
  uint8_t* epi = ring + BD_STAGES * BD_A_BYTES;         // store staging
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + BD_EPI_BYTES);
  uint64_t* empty = full + BD_STAGES;
  uint64_t* tfull = empty + BD_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* gfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int s = blockIdx.x / args.chunks, chunk = blockIdx.x % args.chunks;
  const int t0 = chunk * args.per;
  const int t1 = t0 + args.per < args.m_tiles ? t0 + args.per : args.m_tiles;
  constexpr int KB = BN / BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < BD_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    mbar_init(gfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
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

  if (warp == 0) {
    if (lane == 0) {
      // G[s] once: KB chunks of 64 K-rows (MN-major: BN/64 atoms each) or of
      // 64 K-cols x BN rows (K-major, i.e. G[s]^T)
      mbar_expect_tx(gfull, CF::B_BYTES);
#pragma unroll
      for (int kc = 0; kc < KB; ++kc) {
        uint8_t* dst = sg + kc * (BN * BK * 2);
        if constexpr (B_MN) {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(dst + j * (BK * 128), &map_g, gfull, j * 64, s * BN + kc * BK);
        } else {
          tma_load_2d(dst, &map_g, gfull, kc * BK, s * BN);
        }
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t0; t < t1; ++t) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], BD_A_BYTES);
          tma_load_2d(ring + stage * BD_A_BYTES, &map_x, &full[stage], s * BN + kb * BK, t * BM);
          if (++stage == BD_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(BM, BN, false, B_MN);
    mbar_wait(gfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t g_addr = smem_u32(sg);
    for (int t = t0; t < t1; ++t) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[stage], phase);
        fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(ring + stage * BD_A_BYTES);
          const uint32_t b_addr = g_addr + kb * (BN * BK * 2);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(tmem_d, operand_desc<false>(a_addr, k), operand_desc<B_MN>(b_addr, k), idesc,
                      (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (kb == KB - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == BD_STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    uint8_t* stg = epi + ew * (BD_EPI_BUFS * 32 * 128);
    int acc = 0, buf = 0;
    uint32_t acc_phase = 0;
    for (int t = t0; t < t1; ++t) {
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
#pragma unroll 1
      for (int c = 0; c < BN; c += 64) {
        uint32_t r0[32], r1[32];
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c;
        tmem_ld32(taddr, r0);
        tmem_ld32(taddr + 32, r1);
        if (lane == 0) bulk_wait_read<BD_EPI_BUFS - 1>();  // staging buffer `buf` free again
        __syncwarp();
        uint8_t* row = stg + buf * (32 * 128) + lane * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t* src = q < 4 ? r0 + 8 * q : r1 + 8 * (q - 4);
          uint4 v;
          v.x = pack_bf16(src[0], src[1]);
          v.y = pack_bf16(src[2], src[3]);
          v.z = pack_bf16(src[4], src[5]);
          v.w = pack_bf16(src[6], src[7]);
          *reinterpret_cast<uint4*>(row + ((q ^ (lane & 7)) * 16)) = v;
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&map_y, stg + buf * (32 * 128), s * BN + c, t * BM + ew * 32);
          bulk_commit();
        }
        if (++buf == BD_EPI_BUFS) buf = 0;
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();
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

template <int BN, bool B_MN>
int bd_launch(const CUtensorMap& mx, const CUtensorMap& mg, const CUtensorMap& my, BdArgs a,
              int nb, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(bd_kernel<BN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         BdCfg<BN>::SMEM);
    attr = true;
  }
  void* tok = prof_begin(st);
  bd_kernel<BN, B_MN><<<nb * a.chunks, BD_THREADS, BdCfg<BN>::SMEM, st>>>(mx, mg, my, a);
  prof_end(tok, "tc_blockdiag", 2.0 * a.T * static_cast<double>(nb) * BN * BN, st);
  POETX_LAUNCHED("tc_blockdiag");
  return POETX_OK;
}

}  // namespace
}  // namespace tc

// y = x blockdiag(G) (transpose: G^T) for BF16 x [T, nb*b], G [nb, b, b]
int tc_blockdiag_apply(int64_t T, int64_t nb, int64_t b, const void* g, int transpose,
                       const void* x, void* y, cudaStream_t st) {
  using namespace tc;
  if (!(b == 64 || b == 128 || b == 256) || T <= 0 || nb <= 0) return POETX_ENOTSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
       reinterpret_cast<uintptr_t>(g)) & 15)
    return POETX_ENOTSUPPORTED;
  const int64_t dim = nb * b;
  if (T > INT32_MAX || dim > INT32_MAX) return POETX_ENOTSUPPORTED;
  CUtensorMap mx, mg, my;
  POETX_TRY(make_map(&mx, x, dim, T, dim, 64, BM));
  if (!transpose)
    POETX_TRY(make_map(&mg, g, b, nb * b, b, 64, BK));  // MN-major atoms {64 n, 64 k}
  else
    POETX_TRY(make_map(&mg, g, b, nb * b, b, 64, static_cast<uint32_t>(b)));  // K-major {64 k, b n}
  POETX_TRY(make_map(&my, y, dim, T, dim, 64, 32));
  BdArgs a{};
  a.T = static_cast<int>(T);
  a.b = static_cast<int>(b);
  a.m_tiles = static_cast<int>((T + BM - 1) / BM);
  // one wave: at most (CTAs resident per SM by shared memory) x SMs, so no
  // straggler second wave (b = 256, nb = 22: 154 CTAs -> 132, 44 -> 37.5 us)
  const int smem = b == 256 ? BdCfg<256>::SMEM : b == 128 ? BdCfg<128>::SMEM : BdCfg<64>::SMEM;
  int per_sm = (227 * 1024) / (smem + 1024);
  if (per_sm < 1) per_sm = 1;
  int chunks = static_cast<int>(static_cast<int64_t>(num_sms()) * per_sm / nb);
  if (chunks > a.m_tiles) chunks = a.m_tiles;
  if (chunks < 1) chunks = 1;
  a.per = (a.m_tiles + chunks - 1) / chunks;
  a.chunks = (a.m_tiles + a.per - 1) / a.per;
  const int n = static_cast<int>(nb);
  if (b == 256) return transpose ? bd_launch<256, false>(mx, mg, my, a, n, st) : bd_launch<256, true>(mx, mg, my, a, n, st);
  if (b == 128) return transpose ? bd_launch<128, false>(mx, mg, my, a, n, st) : bd_launch<128, true>(mx, mg, my, a, n, st);
  return transpose ? bd_launch<64, false>(mx, mg, my, a, n, st) : bd_launch<64, true>(mx, mg, my, a, n, st);
}

}  // namespace poetx
