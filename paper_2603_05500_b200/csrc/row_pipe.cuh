// Pair-interleaved persistent row kernels (row_pipe.cu): each entry returns
// POETX_ENOTSUPPORTED_ROW when a shape / alignment does not fit the
// pipelined kernel, and the caller uses the simple staged kernel instead.
#pragma once

#include "common.cuh"

namespace poetx {

constexpr int POETX_ENOTSUPPORTED_ROW = -101;

struct DuPtrs {
  const void* p[3];
};

int rowpipe_rmsnorm_gather_bwd(int64_t T, int64_t d, const void* x, const float* w, const float* rstd, int K,
                               const int32_t* const* inv, const void* const* du, const void* dres, void* dx,
                               float* part, size_t part_rows, int* grid_out, cudaStream_t st);

}  // namespace poetx
