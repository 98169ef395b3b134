// POET-XQ: per-row symmetric int8 storage of the frozen weight (quant.py:
// 22-74).  Row i: scale = absmax_i / 127 (1.0 for an all-zero
// row), code = clip(rint(w / scale), -127, 127) with round-half-to-even, all
// in float64 exactly as the reference does before the scale is stored in
// the layer's float type -- so codes and scales are bit-exact.  Per-row
// scales ride with their rows under gathers, so the premerged copy is the
// quantized base gathered in the quantized domain (quant.py:63-74).
//
// On the device the frozen weight stays int8 (half the bf16 HBM); a layer
// call dequantizes its premerged rows into a transient scratch right before
// the mm2 / adjoint GEMM (one layer at a time), the bf16 analogue of the
// reference's row/column dequantisation inside _mm2 / _mm2_adjoint.
#include "common.cuh"

namespace poetx {
namespace {

template <typename T> __device__ __forceinline__ double to_d(T v) { return static_cast<double>(v); }
template <> __device__ __forceinline__ double to_d(__nv_bfloat16 v) { return static_cast<double>(__bfloat162float(v)); }

// one CTA per row: float64 absmax, then codes
template <typename T, typename S>
__global__ void __launch_bounds__(256) quantize_rows_kernel(int64_t rows, int64_t cols, const T* __restrict__ w,
                                                            int8_t* __restrict__ codes, S* __restrict__ scales) {
  __shared__ double red[8];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const T* row = w + r * cols;
    double mx = 0.0;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmax(mx, fabs(to_d(row[j])));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = mx;
    __syncthreads();
    double amax = 0.0;
    for (int k = 0; k < 8; ++k) amax = fmax(amax, red[k]);
    const double scale = amax > 0.0 ? amax / 127.0 : 1.0;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
      double q = rint(to_d(row[j]) / scale);  // round half to even (np.rint)
      q = fmin(fmax(q, -127.0), 127.0);
      codes[r * cols + j] = static_cast<int8_t>(q);
    }
    if (threadIdx.x == 0) scales[r] = static_cast<S>(scale);
    __syncthreads();
  }
}

template <typename S, typename O>
__device__ __forceinline__ O dq(int8_t c, S s);
template <> __device__ __forceinline__ float dq<float, float>(int8_t c, float s) { return static_cast<float>(c) * s; }
template <> __device__ __forceinline__ double dq<double, double>(int8_t c, double s) { return static_cast<double>(c) * s; }
template <> __device__ __forceinline__ __nv_bfloat16 dq<float, __nv_bfloat16>(int8_t c, float s) {
  return __float2bfloat16_rn(static_cast<float>(c) * s);
}

// out[i, j] = codes[ri(i), ci(j)] * scales[ri(i)]   (gathers optional)
template <typename S, typename O>
__global__ void __launch_bounds__(256) dequant_rows_kernel(int64_t rows, int64_t cols, int64_t ld, const int8_t* __restrict__ codes,
                                                           const S* __restrict__ scales, const int32_t* __restrict__ ri,
                                                           const int32_t* __restrict__ ci, O* __restrict__ out) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t src = ri ? ri[r] : r;
    const int8_t* crow = codes + src * ld;
    const S s = scales[src];
    O* orow = out + r * cols;
    if (!ci && cols % 16 == 0 && ld % 16 == 0) {
      for (int64_t j = threadIdx.x * 16; j < cols; j += blockDim.x * 16) {
        const int4 v = __ldcs(reinterpret_cast<const int4*>(crow + j));
        const int8_t* c = reinterpret_cast<const int8_t*>(&v);
        __align__(16) O o[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) o[q] = dq<S, O>(c[q], s);
        // 16 outputs = 32 / 64 / 128 bytes: whole 16-byte vector stores
        const uint4* src = reinterpret_cast<const uint4*>(o);
        uint4* dst = reinterpret_cast<uint4*>(orow + j);
#pragma unroll
        for (int q = 0; q < static_cast<int>(sizeof(O)) ; ++q) dst[q] = src[q];
      }
    } else {
      for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) orow[j] = dq<S, O>(crow[ci ? ci[j] : j], s);
    }
  }
}

// quantized-domain gather: codes_out[i, j] = codes[ri(i), ci(j)], scales_out[i] = scales[ri(i)]
template <typename S>
__global__ void __launch_bounds__(256) quant_gather_kernel(int64_t rows, int64_t cols, int64_t ld, const int32_t* __restrict__ ri,
                                                           const int32_t* __restrict__ ci, const int8_t* __restrict__ codes,
                                                           const S* __restrict__ scales, int8_t* __restrict__ codes_out,
                                                           S* __restrict__ scales_out) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t src = ri ? ri[r] : r;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
      codes_out[r * cols + j] = codes[src * ld + (ci ? ci[j] : j)];
    if (threadIdx.x == 0) scales_out[r] = scales[src];
  }
}

unsigned row_grid(int64_t rows) { return static_cast<unsigned>(rows < 148 * 16 ? (rows > 0 ? rows : 1) : 148 * 16); }

}  // namespace

int quant_dequant(int dt, int64_t rows, int64_t cols, const int8_t* codes, const void* scales,
                  const int32_t* ri, const int32_t* ci, void* out, cudaStream_t st, int64_t ld) {
  if (ld <= 0) ld = cols;
  if (rows <= 0 || cols <= 0) return POETX_OK;
  switch (dt) {
    case POETX_F32:
      dequant_rows_kernel<float, float><<<row_grid(rows), 256, 0, st>>>(
          rows, cols, ld, codes, static_cast<const float*>(scales), ri, ci, static_cast<float*>(out));
      break;
    case POETX_F64:
      dequant_rows_kernel<double, double><<<row_grid(rows), 256, 0, st>>>(
          rows, cols, ld, codes, static_cast<const double*>(scales), ri, ci, static_cast<double*>(out));
      break;
    case POETX_BF16:
      dequant_rows_kernel<float, __nv_bfloat16><<<row_grid(rows), 256, 0, st>>>(
          rows, cols, ld, codes, static_cast<const float*>(scales), ri, ci, static_cast<__nv_bfloat16*>(out));
      break;
    default:
      set_error("dequantize_rows: unsupported dtype %d", dt);
      return POETX_ESHAPE;
  }
  POETX_LAUNCHED("dequant_rows");
  return POETX_OK;
}

int quant_rows(int dt, int64_t rows, int64_t cols, const void* w, int8_t* codes, void* scales, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return POETX_OK;
  switch (dt) {
    case POETX_F32:
      quantize_rows_kernel<float, float><<<row_grid(rows), 256, 0, st>>>(
          rows, cols, static_cast<const float*>(w), codes, static_cast<float*>(scales));
      break;
    case POETX_F64:
      quantize_rows_kernel<double, double><<<row_grid(rows), 256, 0, st>>>(
          rows, cols, static_cast<const double*>(w), codes, static_cast<double*>(scales));
      break;
    case POETX_BF16:
      quantize_rows_kernel<__nv_bfloat16, float><<<row_grid(rows), 256, 0, st>>>(
          rows, cols, static_cast<const __nv_bfloat16*>(w), codes, static_cast<float*>(scales));
      break;
    default:
      set_error("quantize_rows: unsupported dtype %d", dt);
      return POETX_ESHAPE;
  }
  POETX_LAUNCHED("quantize_rows");
  return POETX_OK;
}

int quant_gather(int dt, int64_t rows, int64_t cols, const int32_t* ri, const int32_t* ci, const int8_t* codes,
                 const void* scales, int8_t* codes_out, void* scales_out, cudaStream_t st, int64_t ld) {
  if (rows <= 0 || cols <= 0) return POETX_OK;
  if (ld <= 0) ld = cols;
  if (param_dtype(dt) == POETX_F64)
    quant_gather_kernel<double><<<row_grid(rows), 256, 0, st>>>(rows, cols, ld, ri, ci, codes,
                                                                 static_cast<const double*>(scales), codes_out,
                                                                 static_cast<double*>(scales_out));
  else
    quant_gather_kernel<float><<<row_grid(rows), 256, 0, st>>>(rows, cols, ld, ri, ci, codes,
                                                                static_cast<const float*>(scales), codes_out,
                                                                static_cast<float*>(scales_out));
  POETX_LAUNCHED("quant_gather");
  return POETX_OK;
}

}  // namespace poetx

using namespace poetx;

extern "C" {

int poetx_quantize_rows(int dtype, int64_t rows, int64_t cols, const void* w, int8_t* codes, void* scales,
                        void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "quantize_rows: unsupported dtype %d", dtype);
  POETX_REQUIRE(rows >= 0 && cols >= 0 && (rows == 0 || cols == 0 || (w && codes && scales)), POETX_ESHAPE,
                "quantize_rows: bad arguments");
  return quant_rows(dtype, rows, cols, w, codes, scales, as_stream(stream));
}

int poetx_dequantize_rows(int dtype, int64_t rows, int64_t cols, int64_t src_cols, const int8_t* codes,
                          const void* scales, const int32_t* row_idx, const int32_t* col_idx, void* out,
                          void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "dequantize_rows: unsupported dtype %d", dtype);
  POETX_REQUIRE(rows >= 0 && cols >= 0 && (rows == 0 || cols == 0 || (codes && scales && out)), POETX_ESHAPE,
                "dequantize_rows: bad arguments");
  return quant_dequant(dtype, rows, cols, codes, scales, row_idx, col_idx, out, as_stream(stream), src_cols);
}

int poetx_quant_gather(int dtype, int64_t rows, int64_t cols, int64_t src_cols, const int32_t* row_idx,
                       const int32_t* col_idx, const int8_t* codes, const void* scales, int8_t* codes_out,
                       void* scales_out, void* stream) {
  POETX_REQUIRE(valid_dtype(dtype), POETX_ESHAPE, "quant_gather: unsupported dtype %d", dtype);
  return quant_gather(dtype, rows, cols, row_idx, col_idx, codes, scales, codes_out, scales_out, as_stream(stream),
                      src_cols);
}

}  // extern "C"
