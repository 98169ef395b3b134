// tcgen05 kernels -- placeholder until the TMA/TMEM GEMM lands.
#include "tc_gemm.cuh"

namespace poetx {

static int g_tc_on = 1;
bool tc_enabled() { return g_tc_on != 0; }

int tc_matmul(int64_t, int64_t, int64_t, const void*, int64_t, int, const void*, int64_t, int,
              void*, int64_t, cudaStream_t) {
  return POETX_ENOTSUPPORTED;
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
