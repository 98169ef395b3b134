// Generic strided, batched SIMT GEMM (CUDA cores).
//
// Used for the fp32 / fp64 parity path (Blackwell has no fp32/fp64 tensor
// core MMA that meets the reference's 1e-5 tolerance: TF32 is ~1e-3) and
// as the fallback for BF16 shapes the tcgen05 kernel does not tile.
// Any operand may be addressed with arbitrary (batch, row, col) strides,
// which is how transposes, block-diagonal segments and the segmented outer
// product are expressed without copies.
#pragma once

#include "common.cuh"

namespace poetx {

struct GemmDesc {
  int64_t M, N, K, batch;
  const void* A; int64_t sAb, sAm, sAk;
  const void* B; int64_t sBb, sBk, sBn;
  void* C;       int64_t sCb, sCm, sCn;
  double alpha;  // C = alpha * (A B) + beta * C
  double beta;
};

constexpr int kSimtBM = 64, kSimtBN = 64, kSimtBK = 16, kSimtThreads = 256;

// 4 consecutive accumulators of a shared row (16-byte aligned): one vector load
template <typename Acc>
__device__ __forceinline__ void ld4(const Acc* p, Acc (&v)[4]) {
  if constexpr (sizeof(Acc) == 4) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
    const double2 x = *reinterpret_cast<const double2*>(p), y = *reinterpret_cast<const double2*>(p + 2);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
  }
}

// 64 x 64 output tile, 256 threads, each a 4 x 4 block of CONSECUTIVE rows and
// columns, so a k step reads its 4 + 4 operands with two vector shared loads
// (the old strided mapping needed eight scalar ones per 16 FMAs); next
// k-tile's global loads are held in registers while the current one computes.
template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(kSimtThreads) simt_gemm_kernel(GemmDesc d) {
  using Acc = typename AccOf<TC>::type;
  constexpr int PAD = 16 / sizeof(Acc);  // rows stay 16-byte aligned
  __shared__ __align__(16) Acc As[kSimtBK][kSimtBM + PAD];
  __shared__ __align__(16) Acc Bs[kSimtBK][kSimtBN + PAD];

  const int64_t bz = blockIdx.z;
  const TA* A = static_cast<const TA*>(d.A) + bz * d.sAb;
  const TB* B = static_cast<const TB*>(d.B) + bz * d.sBb;
  TC* C = static_cast<TC*>(d.C) + bz * d.sCb;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kSimtBM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * kSimtBN;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // rows 4ty.., columns 4tx..

  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = Acc(0);

  // element e of a 64 x 16 tile: consecutive threads walk the contiguous index
  auto a_idx = [&](int e, int& am, int& ak) {
    if (d.sAm == 1) { am = e % kSimtBM; ak = e / kSimtBM; } else { ak = e % kSimtBK; am = e / kSimtBK; }
  };
  auto b_idx = [&](int e, int& bk, int& bn) {
    if (d.sBn == 1) { bn = e % kSimtBN; bk = e / kSimtBN; } else { bk = e % kSimtBK; bn = e / kSimtBK; }
  };
  Acc ra[4], rb[4];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * kSimtThreads;  // 0..1023
      int am, ak, bk, bn;
      a_idx(e, am, ak);
      b_idx(e, bk, bn);
      const int64_t gm = m0 + am, gk = k0 + ak, gn = n0 + bn, gk2 = k0 + bk;
      ra[r] = (gm < d.M && gk < d.K) ? Conv<TA>::to_f(A[gm * d.sAm + gk * d.sAk]) : Acc(0);
      rb[r] = (gn < d.N && gk2 < d.K) ? Conv<TB>::to_f(B[gk2 * d.sBk + gn * d.sBn]) : Acc(0);
    }
  };
  // k-tiles are visited in ascending order and, inside a tile, k ascends:
  // every output element accumulates over k in the same fixed order.
  if (d.K > 0) fetch(0);
  for (int64_t k0 = 0; k0 < d.K; k0 += kSimtBK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * kSimtThreads;
      int am, ak, bk, bn;
      a_idx(e, am, ak);
      b_idx(e, bk, bn);
      As[ak][am] = ra[r];
      Bs[bk][bn] = rb[r];
    }
    __syncthreads();
    if (k0 + kSimtBK < d.K) fetch(k0 + kSimtBK);
#pragma unroll
    for (int kk = 0; kk < kSimtBK; ++kk) {
      Acc a[4], b[4];
      ld4(&As[kk][4 * ty], a);
      ld4(&Bs[kk][4 * tx], b);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }

  const Acc alpha = static_cast<Acc>(d.alpha), beta = static_cast<Acc>(d.beta);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + 4 * ty + i;
    if (gm >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + 4 * tx + j;
      if (gn >= d.N) continue;
      TC* c = C + gm * d.sCm + gn * d.sCn;
      Acc r = acc[i][j];
      if (alpha != Acc(1)) r = alpha * r;
      if (beta != Acc(0)) r = r + beta * Conv<TC>::to_f(*c);
      *c = Conv<TC>::from_f(r);
    }
  }
}

template <typename TA, typename TB, typename TC>
int simt_gemm(const GemmDesc& d, cudaStream_t st) {
  if (d.M <= 0 || d.N <= 0 || d.batch <= 0) return POETX_OK;
  POETX_REQUIRE(d.batch <= 65535, POETX_ESHAPE, "gemm batch %lld too large", (long long)d.batch);
  if (d.K <= 0) {
    // empty contraction: C = beta * C (alpha * 0)
    GemmDesc z = d;
    (void)z;
  }
  dim3 grid(static_cast<unsigned>((d.N + kSimtBN - 1) / kSimtBN),
            static_cast<unsigned>((d.M + kSimtBM - 1) / kSimtBM), static_cast<unsigned>(d.batch));
  POETX_REQUIRE(grid.y <= 65535, POETX_ESHAPE, "gemm M %lld too large", (long long)d.M);
  simt_gemm_kernel<TA, TB, TC><<<grid, kSimtThreads, 0, st>>>(d);
  POETX_LAUNCHED("simt_gemm");
  return POETX_OK;
}

}  // namespace poetx
