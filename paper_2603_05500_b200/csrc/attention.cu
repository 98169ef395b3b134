// Causal self-attention backward for the decoder blocks of Llama-60M/350M/1B
// (sequence 256, head_dim 64, bf16, token-major [B*S, H*hd] tensors as the
// trainer's fused blocks hold them).  The forward stays on cuDNN (its
// natural-log logsumexp [B, H, S] is this kernel's input); cuDNN's backward at
// this shape runs three kernels (dot(dO, O), the flash backward, an fp32 ->
// bf16 dQ conversion) at ~7% of the tensor peak.
//
// One CTA per (batch, head) holds the whole sequence: Q, K, V, dO, O (5 x 32
// KB) in shared memory, and every accumulator in its 512 TMEM columns:
//     S^T, dP^T   128 + 128 columns (key rows x query columns, one tile pair)
//     dV, dK      64 + 64          (key rows; drained after each key tile)
//     dQ[0], dQ[1] 64 + 64         (query rows, accumulated over key tiles)
// so dQ needs no atomics and the result is deterministic.  Tile pairs (key
// tile kt, query tile qt) in causal order: (0,0), (0,1), (1,1).  Per pair:
//     S^T = K_kt Q_qt^T, dP^T = V_kt dO_qt^T                 (tcgen05, K = 64)
//     P^T = exp(scale S^T - lse), dS^T = P^T (dP^T - D)      (epilogue warps)
//     dV += P^T dO_qt, dK += dS^T Q_qt, dQ_qt += dS K_kt     (tcgen05, K = 128)
// with D = rowsum(dO * O) computed from the staged tiles, and scale applied
// to dK and dQ in the drain.  Warp 0 issues the TMA loads, warp 1 the MMAs,
// warps 4..19 (one key / query row per thread = one TMEM lane, four warps per
// lane group splitting the columns) the softmax algebra and the drains.
#include "tc_common.cuh"

namespace poetx {
namespace attn {
using namespace tc;

constexpr int SEQ = 256, HD = 64;
constexpr int TILE = 128 * 128;            // [128 rows x 64 bf16] SW128 block
constexpr int MAT = 2 * TILE;              // 256 rows
constexpr int OFF_Q = 0, OFF_K = MAT, OFF_V = 2 * MAT, OFF_DO = 3 * MAT, OFF_O = 4 * MAT;
constexpr int OFF_PT = OFF_O;              // P^T overwrites O once D is computed
constexpr int OFF_DST = 5 * MAT;
constexpr int OFF_LSE = 6 * MAT, OFF_D = OFF_LSE + SEQ * 4, OFF_BAR = OFF_D + SEQ * 4;
constexpr int SMEM = OFF_BAR + 128 + 1024;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void named_sync_epi() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

__device__ __forceinline__ void unpack_bf16x8(const uint4 u, float (&o)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __bfloat1622float2(h[q]);
    o[2 * q] = f.x;
    o[2 * q + 1] = f.y;
  }
}

// swizzled 16-byte chunk c of row r inside a [rows x 64 bf16] SW128 block
__device__ __forceinline__ uint32_t sw_off(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 16 fp32 TMEM columns of this thread's lane -> 32 bytes of a bf16 row in global
__device__ __forceinline__ void drain_row(uint32_t taddr, float mul, __nv_bfloat16* dst) {
  uint32_t r[16];
  tmem_ld16(taddr, r);
  uint4* out = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    uint4 v;
    v.x = pack_bf16(__float_as_uint(__uint_as_float(r[8 * q + 0]) * mul), __float_as_uint(__uint_as_float(r[8 * q + 1]) * mul));
    v.y = pack_bf16(__float_as_uint(__uint_as_float(r[8 * q + 2]) * mul), __float_as_uint(__uint_as_float(r[8 * q + 3]) * mul));
    v.z = pack_bf16(__float_as_uint(__uint_as_float(r[8 * q + 4]) * mul), __float_as_uint(__uint_as_float(r[8 * q + 5]) * mul));
    v.w = pack_bf16(__float_as_uint(__uint_as_float(r[8 * q + 6]) * mul), __float_as_uint(__uint_as_float(r[8 * q + 7]) * mul));
    out[q] = v;
  }
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 pack_f8(const float* v) {
  uint4 u;
  u.x = pack_bf16(__float_as_uint(v[0]), __float_as_uint(v[1]));
  u.y = pack_bf16(__float_as_uint(v[2]), __float_as_uint(v[3]));
  u.z = pack_bf16(__float_as_uint(v[4]), __float_as_uint(v[5]));
  u.w = pack_bf16(__float_as_uint(v[6]), __float_as_uint(v[7]));
  return u;
}

constexpr int NQ = 4;                  // softmax warps per TMEM lane group (each: 128 / NQ columns)
constexpr int EPI = 128 * NQ;          // warps 4..4+4*NQ-1: softmax algebra and drains
constexpr int THREADS = 128 + EPI;     // warps 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle

__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                    const __grid_constant__ CUtensorMap mo, const float* __restrict__ lse,
                    __nv_bfloat16* __restrict__ dq, __nv_bfloat16* __restrict__ dk,
                    __nv_bfloat16* __restrict__ dv, int H, int64_t ld, float scale) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = /* 1024-byte aligned, kept in the shared address space (STS/LDS) */ smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t *s_full = bars + 1, *p_full = bars + 2, *acc_full = bars + 3, *acc_empty = bars + 4, *fin = bars + 5;
  uint64_t* ldb = bars + 8;  // 4 load stages: dO+O (for D), K0 V0 Q0, Q1, K1 V1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  float* lse_s = reinterpret_cast<float*>(sm + OFF_LSE);
  float* d_s = reinterpret_cast<float*>(sm + OFF_D);
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int row0 = b * SEQ, col0 = h * HD;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&ldb[i], 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, EPI);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, EPI);
    mbar_init(fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // issue order = need order: D's inputs, then the tiles of pair (0,0),
      // then Q1 for (0,1), then K1 V1 for (1,1)
      mbar_expect_tx(&ldb[0], 2 * MAT);
      mbar_expect_tx(&ldb[1], 3 * TILE);
      mbar_expect_tx(&ldb[2], TILE);
      mbar_expect_tx(&ldb[3], 2 * TILE);
      for (int half = 0; half < 2; ++half) {
        tma_load_2d(sm + OFF_DO + half * TILE, &mdo, &ldb[0], col0, row0 + half * 128);
        tma_load_2d(sm + OFF_O + half * TILE, &mo, &ldb[0], col0, row0 + half * 128);
      }
      tma_load_2d(sm + OFF_K, &mk, &ldb[1], col0, row0);
      tma_load_2d(sm + OFF_V, &mv, &ldb[1], col0, row0);
      tma_load_2d(sm + OFF_Q, &mq, &ldb[1], col0, row0);
      tma_load_2d(sm + OFF_Q + TILE, &mq, &ldb[2], col0, row0 + 128);
      tma_load_2d(sm + OFF_K + TILE, &mk, &ldb[3], col0, row0 + 128);
      tma_load_2d(sm + OFF_V + TILE, &mv, &ldb[3], col0, row0 + 128);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t base = smem_u32(sm);
      constexpr uint32_t id_s = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_kv = idesc_bf16(128, 64, false, true);
      constexpr uint32_t id_q = idesc_bf16(128, 64, true, true);
#pragma unroll 1
      for (int it = 0; it < 3; ++it) {
        const int kt = it == 2 ? 1 : 0, qt = it == 0 ? 0 : 1;
        if (it == 0) {
          mbar_wait(&ldb[0], 0);
          mbar_wait(&ldb[1], 0);
        }
        mbar_wait(&ldb[it + 1], 0);
        fence_after();
        // S^T = K_kt Q_qt^T ; dP^T = V_kt dO_qt^T   (K = head_dim)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_bf16(tmem, sdesc(base + OFF_K + kt * TILE + ks * 32, 16, 1024),
                    sdesc(base + OFF_Q + qt * TILE + ks * 32, 16, 1024), id_s, ks > 0);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_bf16(tmem + 128, sdesc(base + OFF_V + kt * TILE + ks * 32, 16, 1024),
                    sdesc(base + OFF_DO + qt * TILE + ks * 32, 16, 1024), id_s, ks > 0);
        umma_commit(s_full);
        mbar_wait(p_full, it & 1);
        fence_after();
        if (it == 2) {
          mbar_wait(acc_empty, 0);
          fence_after();
        }
        const bool first_kv = it != 1, first_q = it != 2;
        // dV += P^T dO_qt ; dK += dS^T Q_qt   (K = 128 queries)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16(tmem + 256, sdesc(base + OFF_PT + (ks / 4) * TILE + (ks % 4) * 32, 16, 1024),
                    sdesc(base + OFF_DO + qt * TILE + ks * 2048, TILE, 1024), id_kv, !(first_kv && ks == 0));
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16(tmem + 320, sdesc(base + OFF_DST + (ks / 4) * TILE + (ks % 4) * 32, 16, 1024),
                    sdesc(base + OFF_Q + qt * TILE + ks * 2048, TILE, 1024), id_kv, !(first_kv && ks == 0));
        // dQ_qt += dS K_kt   (A = dS^T tile read MN-major, K = 128 keys)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16(tmem + 384 + qt * 64, sdesc(base + OFF_DST + ks * 2048, TILE, 1024),
                    sdesc(base + OFF_K + kt * TILE + ks * 2048, TILE, 1024), id_q, !(first_q && ks == 0));
        if (it == 1) umma_commit(acc_full);
      }
      umma_commit(fin);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // warp 4+w: TMEM lanes 32*(w%4).., query / hd column half w/4
    const int lg = (warp - 4) % 4, ch = (warp - 4) / 4;
    const int e = lg * 32 + lane;  // key (or query) row within a tile = TMEM lane
    const int et = threadIdx.x - 128;
    for (int i = et; i < SEQ; i += EPI) lse_s[i] = lse[static_cast<int64_t>(bh) * SEQ + i] * LOG2E;
    mbar_wait(&ldb[0], 0);
    if (et < SEQ) {  // D[q] = sum_c dO[q, c] O[q, c]
      const int q = et, r = q % 128;
      const uint8_t* pd = sm + OFF_DO + (q / 128) * TILE;
      const uint8_t* po = sm + OFF_O + (q / 128) * TILE;
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float a[8], o[8];
        unpack_bf16x8(*reinterpret_cast<const uint4*>(pd + sw_off(r, c)), a);
        unpack_bf16x8(*reinterpret_cast<const uint4*>(po + sw_off(r, c)), o);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += a[j] * o[j];
      }
      d_s[q] = acc;
    }
    named_sync_epi();  // D and lse visible; O's region may now take P^T
    const uint32_t tl = tmem + (static_cast<uint32_t>(lg * 32) << 16);
    const float sl2 = scale * LOG2E;
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
      const int kt = it == 2 ? 1 : 0, qt = it == 0 ? 0 : 1;
      const int kk = kt * 128 + e;
      const bool diag = kt == qt;
      mbar_wait(s_full, it & 1);
      fence_after();
#pragma unroll 1
      for (int c0 = ch * (128 / NQ); c0 < (ch + 1) * (128 / NQ); c0 += 16) {
        uint32_t sv[16], dp[16];
        tmem_ld16(tl + c0, sv);
        tmem_ld16(tl + 128 + c0, dp);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float p[8], ds[8];
          const float4* l4 = reinterpret_cast<const float4*>(lse_s + qt * 128 + c0 + 8 * g);
          const float4* d4 = reinterpret_cast<const float4*>(d_s + qt * 128 + c0 + 8 * g);
          const float4 la = l4[0], lb = l4[1], da = d4[0], db = d4[1];
          const float lq[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
          const float dq8[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = 8 * g + u;
            float pj = ex2(__uint_as_float(sv[j]) * sl2 - lq[u]);
            if (diag && kk > qt * 128 + c0 + j) pj = 0.f;
            p[u] = pj;
            ds[u] = pj * (__uint_as_float(dp[j]) - dq8[u]);
          }
          const int j0 = c0 + 8 * g;
          const uint32_t off = (j0 / 64) * TILE + sw_off(e, (j0 % 64) / 8);
          *reinterpret_cast<uint4*>(sm + OFF_PT + off) = pack_f8(p);
          *reinterpret_cast<uint4*>(sm + OFF_DST + off) = pack_f8(ds);
        }
      }
      fence_async_smem();
      fence_before();
      mbar_arrive(p_full);
      if (it == 1) {  // key tile 0 complete: drain dV, dK (this thread: 32 of the 64 columns)
        mbar_wait(acc_full, 0);
        fence_after();
        drain_row(tl + 256 + ch * 16, 1.f, dv + (row0 + e) * ld + col0 + ch * 16);
        drain_row(tl + 320 + ch * 16, scale, dk + (row0 + e) * ld + col0 + ch * 16);
        fence_before();
        mbar_arrive(acc_empty);
      }
    }
    mbar_wait(fin, 0);
    fence_after();
    drain_row(tl + 256 + ch * 16, 1.f, dv + (row0 + 128 + e) * ld + col0 + ch * 16);
    drain_row(tl + 320 + ch * 16, scale, dk + (row0 + 128 + e) * ld + col0 + ch * 16);
    drain_row(tl + 384 + ch * 16, scale, dq + (row0 + e) * ld + col0 + ch * 16);
    drain_row(tl + 448 + ch * 16, scale, dq + (row0 + 128 + e) * ld + col0 + ch * 16);
  }

  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace attn
}  // namespace poetx

using namespace poetx;

extern "C" int poetx_attention_bwd(int64_t B, int64_t S, int64_t H, int64_t hd, const void* q, const void* k,
                                   const void* v, const void* o, const void* dout, const float* lse, void* dq,
                                   void* dk, void* dv, void* stream) {
  POETX_REQUIRE(S == attn::SEQ && hd == attn::HD, POETX_ECONFIG,
                "attention_bwd: only seq %d, head_dim %d (got %lld, %lld)", attn::SEQ, attn::HD, (long long)S,
                (long long)hd);
  POETX_REQUIRE(B > 0 && H > 0 && q && k && v && o && dout && lse && dq && dk && dv, POETX_ESHAPE,
                "attention_bwd: bad arguments");
  const int64_t ld = H * hd;
  for (const void* p : {q, k, v, o, dout, static_cast<const void*>(dq), static_cast<const void*>(dk),
                        static_cast<const void*>(dv)})
    POETX_REQUIRE((reinterpret_cast<uintptr_t>(p) & 15) == 0, POETX_ESHAPE, "attention_bwd: 16-byte alignment");
  CUtensorMap m[5];
  const void* src[5] = {q, k, v, dout, o};
  for (int i = 0; i < 5; ++i) POETX_TRY(tc::make_map(&m[i], src[i], ld, B * S, ld, 64, 128));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::SMEM);
    attr = true;
  }
  attn::attn_bwd_kernel<<<static_cast<unsigned>(B * H), attn::THREADS, attn::SMEM, as_stream(stream)>>>(
      m[0], m[1], m[2], m[3], m[4], lse, static_cast<__nv_bfloat16*>(dq), static_cast<__nv_bfloat16*>(dk),
      static_cast<__nv_bfloat16*>(dv), static_cast<int>(H), ld, 0.125f);
  POETX_LAUNCHED("attention_bwd");
  return POETX_OK;
}
