// Shared plumbing for the poetx_b200 C ABI: status/last-error handling,
// launch accounting, dtype traits.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/poetx_b200.h"

namespace poetx {

void set_error(const char* fmt, ...);
std::atomic<uint64_t>& launch_counter();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Status helpers -------------------------------------------------------------
#define POETX_REQUIRE(cond, code, ...)   \
  do {                                   \
    if (!(cond)) {                       \
      ::poetx::set_error(__VA_ARGS__);   \
      return (code);                     \
    }                                    \
  } while (0)

#define POETX_TRY(expr)          \
  do {                           \
    int _rc = (expr);            \
    if (_rc != POETX_OK) return _rc; \
  } while (0)

inline int check_launch(const char* what) {
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return POETX_ECUDA;
  }
  return POETX_OK;
}
#define POETX_LAUNCHED(name) POETX_TRY(::poetx::check_launch(name))

inline size_t elt_size(int dtype) {
  switch (dtype) {
    case POETX_F32: return 4;
    case POETX_F64: return 8;
    case POETX_BF16: return 2;
  }
  return 0;
}
inline bool valid_dtype(int dtype) { return dtype == POETX_F32 || dtype == POETX_F64 || dtype == POETX_BF16; }
// parameter / factor type for a layer dtype: fp64 layers keep fp64, others fp32
inline int param_dtype(int dtype) { return dtype == POETX_F64 ? POETX_F64 : POETX_F32; }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// bump allocator over a caller-provided workspace
struct Workspace {
  char* base;
  size_t size;
  size_t used = 0;
  Workspace(void* p, size_t n) : base(static_cast<char*>(p)), size(n) {}
  template <typename T>
  T* take(size_t count) {
    size_t bytes = align_up(count * sizeof(T));
    if (used + bytes > size) return nullptr;
    T* r = reinterpret_cast<T*>(base + used);
    used += bytes;
    return r;
  }
  void* take_bytes(size_t bytes) {
    bytes = align_up(bytes);
    if (used + bytes > size) return nullptr;
    void* r = base + used;
    used += bytes;
    return r;
  }
};

// Element conversions ----------------------------------------------------------
template <typename T> struct Conv;
template <> struct Conv<float> {
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct Conv<double> {
  __device__ __forceinline__ static double to_f(double x) { return x; }
  __device__ __forceinline__ static double from_f(double x) { return x; }
};
template <> struct Conv<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

template <typename Src, typename Dst>
__device__ __forceinline__ Dst cvt(Src x) {
  using A = typename AccOf<Dst>::type;
  return Conv<Dst>::from_f(static_cast<A>(Conv<Src>::to_f(x)));
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

}  // namespace poetx
