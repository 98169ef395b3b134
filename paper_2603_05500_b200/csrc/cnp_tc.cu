// Cayley-Neumann parameterization on tensor cores for the BF16 path
// (k = 3, cnp.py:99-145), batched over an arbitrary stack of b x b blocks
// -- in the trainer, every block of every POET-X layer of the model at once,
// because the packed parameters of the whole model are one flat buffer.
//
// Forward (3 launches + 2 elementwise):
//   Q        = unpack(packed)                       -> QQ2[:, :, 0:b]   (bf16)
//   Q^2      = Q Q                      (tcgen05)   -> QQ2[:, :, b:2b]
//   [Q^3|Q^4] = Q^2 [Q | Q^2]           (tcgen05, one N = 2b product)
//   G        = I + 2(Q + Q^2 + Q^3) + Q^4   (fp32 math, reference order) -> bf16 (+fp32)
// QQ2 = [Q | Q^2] is the cache the backward reuses (the paper's
// "load Q and Q^2 once" observation).
//
// Backward (paper's regrouping of the six-product closed form, cnp.py:136-145):
//   N1 = dG ; N2 = -(N1 Q + Q N1)                          (2 tcgen05, fp32 acc)
//   dQ = 2(N1 + N2) + (2Q + Q^2)^T N2 + (2 N1 + N2) (Q^2)^T (2 tcgen05, fp32 acc)
//   packed grad g_ij = dQ_ij - dQ_ji                     (cnp.py:81-86)
// Q^T = -Q and the transposed operands are free: a transpose is the other
// operand major in the UMMA descriptor.
#include "common.cuh"
#include "tc_gemm.cuh"

namespace poetx {

namespace {

__device__ __forceinline__ int64_t pidx(int64_t i, int64_t j, int64_t b) {
  return i * b - i * (i + 1) / 2 + (j - i - 1);
}

// packed fp32 -> Q (bf16) into the left half of QQ2 [nb, b, 2b]
__global__ void unpack_q_kernel(int64_t nb, int64_t b, const float* __restrict__ packed,
                                __nv_bfloat16* __restrict__ qq2) {
  const int64_t pairs = b * (b - 1) / 2, total = nb * b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e / (b * b), r = e % (b * b), i = r / b, j = r % b;
    float v = 0.f;
    if (i < j) v = packed[s * pairs + pidx(i, j, b)];
    else if (i > j) v = -packed[s * pairs + pidx(j, i, b)];
    qq2[(s * b + i) * 2 * b + j] = __float2bfloat16_rn(v);
  }
}

// G = 2 (Q + Q2 + Q3) + Q4 + I  (cnp.py:113-115 operation order)
__global__ void combine_fwd_kernel(int64_t nb, int64_t b, const __nv_bfloat16* __restrict__ qq2,
                                   const __nv_bfloat16* __restrict__ q34,
                                   __nv_bfloat16* __restrict__ g16, float* __restrict__ g32) {
  const int64_t total = nb * b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e / (b * b), r = e % (b * b), i = r / b, j = r % b;
    int64_t row = (s * b + i) * 2 * b;
    float q = __bfloat162float(qq2[row + j]), q2 = __bfloat162float(qq2[row + b + j]);
    float q3 = __bfloat162float(q34[row + j]), q4 = __bfloat162float(q34[row + b + j]);
    float v = 2.f * ((q + q2) + q3) + q4;
    if (i == j) v += 1.f;
    if (g16) g16[e] = __float2bfloat16_rn(v);
    if (g32) g32[e] = v;
  }
}

__global__ void to_bf16_f32_kernel(int64_t total, const float* __restrict__ x,
                                   __nv_bfloat16* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = __float2bfloat16_rn(x[e]);
}

// in place over n2 (becomes dQ's base): base = 2 (N1 + N2); also
// N2 (bf16), R = 2 N1 + N2 (bf16), P = 2 Q + Q^2 (bf16)
__global__ void bwd_prep_kernel(int64_t nb, int64_t b, const float* __restrict__ dg,
                                float* __restrict__ n2_dq, const __nv_bfloat16* __restrict__ qq2,
                                __nv_bfloat16* __restrict__ n2b, __nv_bfloat16* __restrict__ rm,
                                __nv_bfloat16* __restrict__ pm) {
  const int64_t total = nb * b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e / (b * b), r = e % (b * b), i = r / b, j = r % b;
    int64_t row = (s * b + i) * 2 * b;
    float n1 = dg[e], n2 = n2_dq[e];
    n2_dq[e] = 2.f * (n1 + n2);
    n2b[e] = __float2bfloat16_rn(n2);
    rm[e] = __float2bfloat16_rn(2.f * n1 + n2);
    pm[e] = __float2bfloat16_rn(2.f * __bfloat162float(qq2[row + j]) + __bfloat162float(qq2[row + b + j]));
  }
}

__global__ void pack_dq_kernel(int64_t nb, int64_t b, const float* __restrict__ dq,
                               float* __restrict__ g, int accumulate) {
  const int64_t pairs = b * (b - 1) / 2, total = nb * pairs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e / pairs, p = e % pairs;
    // invert the row-major strict-upper-triangle index p -> (i, j)
    int64_t i = static_cast<int64_t>((2.0 * b - 1 - sqrt((2.0 * b - 1) * (2.0 * b - 1) - 8.0 * p)) / 2);
    while (i > 0 && pidx(i, i + 1, b) > p) --i;
    while (pidx(i + 1, i + 2, b) <= p && i + 1 < b - 1) ++i;
    int64_t j = p - pidx(i, i + 1, b) + i + 1;
    const float* blk = dq + s * b * b;
    float v = blk[i * b + j] - blk[j * b + i];
    g[e] = accumulate ? g[e] + v : v;
  }
}

TcProblem stack_problem(int64_t nb, int64_t b, int64_t N, void* C, int64_t ldc, int64_t c_goff,
                        int out_f32, int accumulate, float alpha, const char* name) {
  TcProblem p{};
  p.M = b; p.N = N; p.K = b; p.groups = static_cast<int>(nb); p.splits = 1;
  p.bn = static_cast<int>(N < 256 ? N : 256);
  p.a_g1 = static_cast<int>(b);
  p.b_g1 = static_cast<int>(b);
  p.C = C; p.ldc = ldc; p.c_goff = c_goff;
  p.out_f32 = out_f32; p.accumulate = accumulate; p.alpha = alpha; p.name = name; p.tma_epi = 1;
  return p;
}

int check(int64_t nb, int64_t b) {
  POETX_REQUIRE(nb >= 1 && (b == 64 || b == 128 || b == 256), POETX_ESHAPE,
                "tensor-core CNP needs b in {64, 128, 256}, got %lld", (long long)b);
  POETX_REQUIRE(nb * b < INT32_MAX / 2, POETX_ESHAPE, "tensor-core CNP: stack too large");
  return POETX_OK;
}

}  // namespace
}  // namespace poetx

using namespace poetx;

extern "C" {

size_t poetx_cnp_tc_workspace_bytes(int64_t nb, int64_t b) {
  const size_t blk = static_cast<size_t>(nb * b * b);
  // fwd: Q34 [nb,b,2b] bf16 ; bwd: N1 bf16, N2/dQ fp32, N2 bf16, R bf16, P bf16
  size_t fwd = align_up(blk * 4);
  size_t bwd = align_up(blk * 2) * 4 + align_up(blk * 4);
  return (fwd > bwd ? fwd : bwd) + 4096;
}

int poetx_cnp_forward_tc(int64_t nb, int64_t b, const float* packed, void* qq2, void* g_bf16,
                         float* g_f32, void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check(nb, b));
  POETX_REQUIRE(packed && qq2 && (g_bf16 || g_f32), POETX_ESHAPE, "cnp_forward_tc: null operand");
  cudaStream_t st = as_stream(stream);
  Workspace w(ws, ws_bytes);
  auto* q34 = w.take<__nv_bfloat16>(static_cast<size_t>(nb * b * 2 * b));
  POETX_REQUIRE(q34, POETX_ESHAPE, "cnp_forward_tc: workspace too small");
  auto* QQ2 = static_cast<__nv_bfloat16*>(qq2);
  const int64_t total = nb * b * b;
  unpack_q_kernel<<<grid_for(total, 256), 256, 0, st>>>(nb, b, packed, QQ2);
  POETX_LAUNCHED("cnp_unpack");
  // Q^2 = Q Q : A = Q (K-major), B = Q (MN-major), out -> right half of QQ2
  TcOperand qa{QQ2, nb * b, b, 2 * b, false};
  TcOperand qb{QQ2, nb * b, b, 2 * b, true};
  TcProblem p1 = stack_problem(nb, b, b, QQ2 + b, 2 * b, 2 * b * b, 0, 0, 1.f, "tc_cnp");
  POETX_TRY(tc_grouped(qa, qb, p1, st));
  // [Q^3 | Q^4] = Q^2 [Q | Q^2]
  TcOperand q2a{QQ2 + b, nb * b, b, 2 * b, false};
  TcOperand qqb{QQ2, nb * b, 2 * b, 2 * b, true};
  TcProblem p2 = stack_problem(nb, b, 2 * b, q34, 2 * b, 2 * b * b, 0, 0, 1.f, "tc_cnp");
  POETX_TRY(tc_grouped(q2a, qqb, p2, st));
  combine_fwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(nb, b, QQ2, q34,
                                                           static_cast<__nv_bfloat16*>(g_bf16), g_f32);
  POETX_LAUNCHED("cnp_combine_tc");
  return POETX_OK;
}

int poetx_cnp_backward_tc(int64_t nb, int64_t b, const void* qq2, const float* dg, float* dpacked,
                          int accumulate, void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check(nb, b));
  POETX_REQUIRE(qq2 && dg && dpacked, POETX_ESHAPE, "cnp_backward_tc: null operand");
  cudaStream_t st = as_stream(stream);
  const int64_t total = nb * b * b;
  Workspace w(ws, ws_bytes);
  auto* n1b = w.take<__nv_bfloat16>(total);
  auto* n2b = w.take<__nv_bfloat16>(total);
  auto* rm = w.take<__nv_bfloat16>(total);
  auto* pm = w.take<__nv_bfloat16>(total);
  auto* dq = w.take<float>(total);  // N2, then dQ in place
  POETX_REQUIRE(n1b && n2b && rm && pm && dq, POETX_ESHAPE, "cnp_backward_tc: workspace too small");
  const auto* QQ2 = static_cast<const __nv_bfloat16*>(qq2);
  to_bf16_f32_kernel<<<grid_for(total, 256), 256, 0, st>>>(total, dg, n1b);
  POETX_LAUNCHED("cnp_bwd_cast");
  TcOperand q_k{QQ2, nb * b, b, 2 * b, false};        // Q as K-major A
  TcOperand q_mn{QQ2, nb * b, b, 2 * b, true};        // Q as MN-major B
  TcOperand n1_k{n1b, nb * b, b, b, false};
  TcOperand n1_mn{n1b, nb * b, b, b, true};
  // N2 = -(N1 Q) - (Q N1)
  TcProblem pa = stack_problem(nb, b, b, dq, b, b * b, 1, 0, -1.f, "tc_cnp");
  POETX_TRY(tc_grouped(n1_k, q_mn, pa, st));
  TcProblem pb = stack_problem(nb, b, b, dq, b, b * b, 1, 1, -1.f, "tc_cnp");
  POETX_TRY(tc_grouped(q_k, n1_mn, pb, st));
  bwd_prep_kernel<<<grid_for(total, 256), 256, 0, st>>>(nb, b, dg, dq, QQ2, n2b, rm, pm);
  POETX_LAUNCHED("cnp_bwd_prep");
  // dQ += P^T N2 : A = P^T (MN-major view of P), B = N2 (MN-major)
  TcOperand pt{pm, nb * b, b, b, true};
  TcOperand n2_mn{n2b, nb * b, b, b, true};
  TcProblem pc = stack_problem(nb, b, b, dq, b, b * b, 1, 1, 1.f, "tc_cnp");
  POETX_TRY(tc_grouped(pt, n2_mn, pc, st));
  // dQ += R (Q^2)^T : A = R (K-major), B = (Q^2)^T (K-major view of Q^2)
  TcOperand r_k{rm, nb * b, b, b, false};
  TcOperand q2t{QQ2 + b, nb * b, b, 2 * b, false};
  TcProblem pd = stack_problem(nb, b, b, dq, b, b * b, 1, 1, 1.f, "tc_cnp");
  POETX_TRY(tc_grouped(r_k, q2t, pd, st));
  const int64_t pairs = nb * (b * (b - 1) / 2);
  pack_dq_kernel<<<grid_for(pairs, 256), 256, 0, st>>>(nb, b, dq, dpacked, accumulate);
  POETX_LAUNCHED("cnp_pack_tc");
  return POETX_OK;
}

}  // extern "C"
