// Per-kernel device timing hooks: when enabled, selected launches are
// bracketed by CUDA events recorded on the launching stream, so bench.py
// can report a kernel's average device duration inside a real step.
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace poetx {

struct ProfRec {
  cudaEvent_t start, stop;
  double flops;
};
struct ProfState {
  std::mutex mu;
  bool on = false;
  std::unordered_map<std::string, std::vector<ProfRec>> recs;
  std::vector<cudaEvent_t> pool;
};
static ProfState& prof() {
  static ProfState s;
  return s;
}
bool prof_on() { return prof().on; }

static cudaEvent_t take_event() {
  auto& s = prof();
  if (!s.pool.empty()) {
    cudaEvent_t e = s.pool.back();
    s.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// returns an opaque token; call prof_end after the launch
void* prof_begin(cudaStream_t st) {
  auto& s = prof();
  std::lock_guard<std::mutex> g(s.mu);
  if (!s.on) return nullptr;
  cudaEvent_t e = take_event();
  cudaEventRecord(e, st);
  return reinterpret_cast<void*>(e);
}
void prof_end(void* token, const char* name, double flops, cudaStream_t st) {
  if (!token) return;
  auto& s = prof();
  std::lock_guard<std::mutex> g(s.mu);
  cudaEvent_t e = take_event();
  cudaEventRecord(e, st);
  s.recs[name].push_back({reinterpret_cast<cudaEvent_t>(token), e, flops});
}

}  // namespace poetx

using namespace poetx;

extern "C" {
void poetx_prof_enable(int on) {
  std::lock_guard<std::mutex> g(prof().mu);
  prof().on = on != 0;
}
void poetx_prof_reset(void) {
  auto& s = prof();
  std::lock_guard<std::mutex> g(s.mu);
  for (auto& kv : s.recs)
    for (auto& r : kv.second) {
      s.pool.push_back(r.start);
      s.pool.push_back(r.stop);
    }
  s.recs.clear();
}
int poetx_prof_query(const char* name, double* total_ms, int64_t* count, double* flops) {
  auto& s = prof();
  std::lock_guard<std::mutex> g(s.mu);
  double ms = 0, fl = 0;
  int64_t n = 0;
  auto it = s.recs.find(name ? name : "");
  if (it != s.recs.end()) {
    for (auto& r : it->second) {
      if (cudaEventSynchronize(r.stop) != cudaSuccess) {
        set_error("prof_query: event sync failed");
        return POETX_ECUDA;
      }
      float e = 0;
      cudaEventElapsedTime(&e, r.start, r.stop);
      ms += e;
      fl += r.flops;
      ++n;
    }
  }
  if (total_ms) *total_ms = ms;
  if (count) *count = n;
  if (flops) *flops = fl;
  return POETX_OK;
}
}

// FP32 CUDA-core peak probe (the fp32 parity path's roofline
// denominator).  Every thread runs 8 independent FFMA chains, so the FMA
// pipes, not latency, bound it; FLOP per launch = 2 * 8 * iters * threads.
namespace poetx {
__global__ void __launch_bounds__(256) ffma_probe_kernel(int64_t iters, float* sink) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  const float b = 0.999f, c = 1e-4f;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678f) sink[threadIdx.x] = s;  // keeps the chains live
}
}  // namespace poetx

extern "C" int poetx_ffma_probe(int64_t iters, int64_t ctas, float* sink, double* flops, void* stream) {
  POETX_REQUIRE(iters > 0 && ctas > 0 && sink, POETX_ESHAPE, "ffma_probe: bad arguments");
  poetx::ffma_probe_kernel<<<static_cast<unsigned>(ctas), 256, 0, as_stream(stream)>>>(iters, sink);
  POETX_LAUNCHED("ffma_probe");
  if (flops) *flops = 2.0 * 8.0 * static_cast<double>(iters) * static_cast<double>(ctas) * 256.0;
  return POETX_OK;
}
