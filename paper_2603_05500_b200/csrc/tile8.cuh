// Feature-major 8-token tiles for the feature-permutation kernel (ops.cu):
// a tile of 8 token rows is staged
// TRANSPOSED in shared memory -- one 16-byte slot per feature holding its 8
// token values, XOR-swizzled within groups of 8 so the transposing stores are
// conflict-free -- so gathering feature f for all 8 tokens is ONE 16-byte LDS
// instead of eight conflicted 2-byte LDS.  8x8 bf16 transposes are 32 PRMTs.
// (Measured for RoPE and the residual scatter too: no gain there -- their
// staged kernels already run at 2.4 / 5.8 TB/s -- so only the permute uses it.)
#pragma once

#include <cstdint>

namespace poetx {

// r[row] (8 bf16) -> c[col] (8 bf16): c[col] word i = {row 2i, row 2i+1}
__device__ __forceinline__ void tr8x8(const uint4 (&r)[8], uint4 (&c)[8]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a[4] = {r[2 * i].x, r[2 * i].y, r[2 * i].z, r[2 * i].w};
    const uint32_t b[4] = {r[2 * i + 1].x, r[2 * i + 1].y, r[2 * i + 1].z, r[2 * i + 1].w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      reinterpret_cast<uint32_t*>(&c[2 * w])[i] = __byte_perm(a[w], b[w], 0x5410);
      reinterpret_cast<uint32_t*>(&c[2 * w + 1])[i] = __byte_perm(a[w], b[w], 0x7632);
    }
  }
}
__device__ __forceinline__ int fslot(int f) { return (f & ~7) | ((f ^ (f >> 3)) & 7); }

// stage tokens [r0, r0 + nr) (nr <= 8) of a [T, W] bf16 tensor as W slots
__device__ __forceinline__ void stage_t8(uint4* slots, const __nv_bfloat16* x, int64_t r0, int nr, int W) {
  const int nv = W / 8;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    uint4 rr[8], cc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
      rr[r] = r < nr ? __ldcs(reinterpret_cast<const uint4*>(x + (r0 + r) * W) + c) : make_uint4(0, 0, 0, 0);
    tr8x8(rr, cc);
#pragma unroll
    for (int k = 0; k < 8; ++k) slots[fslot(8 * c + k)] = cc[k];
  }
}

}  // namespace poetx
