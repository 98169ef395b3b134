// tcgen05 / TMEM / TMA tensor-core GEMM for the BF16 path (sm_100a).
//
//   C[M,N] = A[M,K] . op(B)[K,N]     BF16 operands, FP32 accumulation in TMEM
//
// used for the layer's one dense product t = a PM (mm2, layer.py:222) and
// its adjoint da = dt PM^T (layer.py:249).  A is K-major (row-major
// activations); B is MN-major for mm2 (PM row-major [K=m, N=n]) and
// K-major for the adjoint (PM read as [N=m, K=n]), selected by the UMMA
// instruction descriptor -- PM is stored once.
//
// Structure (one CTA per SM, persistent over 128x256 output tiles):
//   warp 0      TMA producer: 4-stage ring of {A 128x64, B 256x64} tiles
//               (SWIZZLE_128B), mbarrier full/empty handshake;
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma
//               (M=128, N=256, K=16) into a double-buffered TMEM
//               accumulator (2 x 256 fp32 columns), tcgen05.commit frees
//               smem stages and publishes finished accumulators;
//   warp 2      TMEM allocator (512 columns);
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> bf16 -> global, then release
//               the accumulator so the next tile's MMAs overlap the store.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "tc_gemm.cuh"

namespace poetx {

void* prof_begin(cudaStream_t st);
void prof_end(void* token, const char* name, double flops, cudaStream_t st);

static int g_tc_on = 1;
bool tc_enabled() { return g_tc_on != 0; }

namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;             // 16 KB
constexpr int B_BYTES = BN * BK * 2;             // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 48 KB
constexpr int TMEM_COLS = 512;                   // 2 accumulators x 256 fp32 columns
constexpr int THREADS = 256;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t spins = 0;
  while (!mbar_try_wait(a, parity)) {
    if (++spins == (1u << 28)) __trap();  // never hang the box: fail loudly
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B (sm100 layout code 2, version 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// instruction descriptor kind::f16: D fp32, A/B bf16, A K-major, B major per flag
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t*>(&v);
}

struct GemmArgs {
  int M, N, K;
  __nv_bfloat16* C;
  int64_t ldc;
  int m_tiles, n_tiles;
};

// ------------------------------------------------------------------ kernel --
template <bool B_MN_MAJOR>
__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_tiles = args.m_tiles * args.n_tiles;
  const int k_blocks = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / args.n_tiles) * BM, n0 = (tile % args.n_tiles) * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sa, &map_a, &full[stage], kb * BK, m0);
          if constexpr (B_MN_MAJOR) {
            // four 64-wide N atoms, each BK K-rows of 128 B
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * (BK * 128), &map_b, &full[stage], n0 + j * 64, kb * BK);
          } else {
            tma_load_2d(sb, &map_b, &full[stage], kb * BK, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = idesc_bf16(BM, BN, B_MN_MAJOR);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major SW128: advance 16 elements = 32 B inside the 128 B swizzle row
            const uint64_t ad = sdesc(a_addr + k * 32, 16, 1024);
            uint64_t bd;
            if constexpr (B_MN_MAJOR)
              bd = sdesc(b_addr + k * 16 * 128, BK * 128, 1024);  // 16 K-rows per step
            else
              bd = sdesc(b_addr + k * 32, 16, 1024);
            umma_bf16(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);  // smem stage free once these MMAs retire
          if (kb == k_blocks - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile / args.n_tiles) * BM, n0 = (tile % args.n_tiles) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      const int row = m0 + ew * 32 + lane;
      __nv_bfloat16* crow = args.C + static_cast<int64_t>(row) * args.ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c, r);
        if (row < args.M && n0 + c < args.N) {
          uint4* dst = reinterpret_cast<uint4*>(crow + n0 + c);
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
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

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

// 2-D bf16 tensor map: dims {inner, outer}, row pitch in elements, box {bi, bo}
int make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch,
             uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  POETX_REQUIRE(fn != nullptr, POETX_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  POETX_REQUIRE(r == CUDA_SUCCESS, POETX_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
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

template <bool MN>
int launch(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc_gemm_kernel<MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES);
    attr_set = true;
  }
  int tiles = a.m_tiles * a.n_tiles;
  int grid = tiles < num_sms() ? tiles : num_sms();
  void* tok = prof_begin(st);
  tc_gemm_kernel<MN><<<grid, THREADS, SMEM_BYTES, st>>>(ma, mb, a);
  prof_end(tok, "tc_gemm", 2.0 * a.M * a.N * a.K, st);
  POETX_LAUNCHED("tc_gemm");
  return POETX_OK;
}

}  // namespace tc

int tc_matmul(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int transA,
              const void* B, int64_t ldb, int transB, void* C, int64_t ldc, cudaStream_t st) {
  using namespace tc;
  if (transA) return POETX_ENOTSUPPORTED;
  if (M <= 0 || N <= 0) return POETX_OK;
  if (K <= 0 || N % 32 || K % 8 || lda % 8 || ldb % 8 || ldc % 8) return POETX_ENOTSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
       reinterpret_cast<uintptr_t>(C)) & 15)
    return POETX_ENOTSUPPORTED;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return POETX_ENOTSUPPORTED;
  CUtensorMap ma, mb;
  POETX_TRY(make_map(&ma, A, K, M, lda, BK, BM));
  GemmArgs a{static_cast<int>(M), static_cast<int>(N), static_cast<int>(K),
             static_cast<__nv_bfloat16*>(C), ldc, static_cast<int>((M + BM - 1) / BM),
             static_cast<int>((N + BN - 1) / BN)};
  if (transB) {
    // B stored [N, K] row-major: K-major operand
    POETX_TRY(make_map(&mb, B, K, N, ldb, BK, BN));
    return launch<false>(ma, mb, a, st);
  }
  // B stored [K, N] row-major: MN-major operand, 64-wide N atoms
  POETX_TRY(make_map(&mb, B, N, K, ldb, 64, BK));
  return launch<true>(ma, mb, a, st);
}

int tc_blockdiag(const GemmDesc&, cudaStream_t) { return POETX_ENOTSUPPORTED; }
size_t tc_outer_ws_bytes(int64_t, int64_t, int64_t) { return 0; }
int tc_segmented_outer(int64_t, int64_t, int64_t, const void*, const void*, float*, Workspace&,
                       cudaStream_t) {
  return POETX_ENOTSUPPORTED;
}

}  // namespace poetx

extern "C" int poetx_tc_enabled(void) { return poetx::g_tc_on; }
extern "C" void poetx_set_tc_enabled(int on) { poetx::g_tc_on = on ? 1 : 0; }
