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

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}
__device__ __forceinline__ uint4 pack_bf8(const float (&v)[8]) {
  return make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]), pack_bf2(v[4], v[5]), pack_bf2(v[6], v[7]));
}
__device__ __forceinline__ void unpack_bf8(const uint4 u, float (&o)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    o[2 * q] = __uint_as_float(w[q] << 16);
    o[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ int64_t pidx(int64_t i, int64_t j, int64_t b) {
  return i * b - i * (i + 1) / 2 + (j - i - 1);
}

// All element-wise CNP kernels work on 64 x 64 tiles of one b x b block
// (b in {64, 128, 256}); a grid-stride loop runs over (block, tile pair).
// The skew structure pairs tile (I, J) with its transpose (J, I), so the
// transposed half goes through shared memory and every global access is a
// contiguous row segment (the packed upper triangle is row-contiguous).
constexpr int TL = 64;

// tile pairs (I <= J) of an nt x nt tile grid, enumerated row-major
__device__ __forceinline__ void tile_pair(int t, int nt, int& I, int& J) {
  I = 0;
  while (t >= nt - I) { t -= nt - I; ++I; }
  J = I + t;
}

// packed fp32 -> Q (bf16) into the left half of QQ2 [nb, b, 2b]
__global__ void __launch_bounds__(256) unpack_q_kernel(int64_t nb, int64_t b, const float* __restrict__ packed,
                                                       __nv_bfloat16* __restrict__ qq2) {
  __shared__ float tile[TL][TL + 1];
  const int nt = static_cast<int>(b / TL), npair = nt * (nt + 1) / 2;
  const int64_t pairs = b * (b - 1) / 2;
  const int tx = threadIdx.x % TL, ty = threadIdx.x / TL;  // 64 x 4
  for (int64_t w = blockIdx.x; w < nb * npair; w += gridDim.x) {
    const int64_t s = w / npair;
    int I, J;
    tile_pair(static_cast<int>(w % npair), nt, I, J);
    const float* pk = packed + s * pairs;
    // upper tile U[i][j] = Q[I*64+i, J*64+j] (strict upper part of a diagonal tile)
    for (int i = ty; i < TL; i += 4) {
      const int64_t gi = I * TL + i, gj = J * TL + tx;
      tile[i][tx] = gj > gi ? pk[pidx(gi, gj, b)] : 0.f;
    }
    __syncthreads();
    __nv_bfloat16* blk = qq2 + s * b * 2 * b;
    // rows of tile (I, J): Q = U ; rows of tile (J, I): Q = -U^T (diagonal tile: both)
    for (int e = threadIdx.x; e < TL * TL / 8; e += 256) {
      const int i = e / 8, c = (e % 8) * 8;
      float u[8], v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float up = tile[i][c + q], lo = tile[c + q][i];
        u[q] = I == J ? (c + q > i ? up : (c + q < i ? -lo : 0.f)) : up;
        v[q] = -lo;
      }
      uint4 pu, pv;
      pu.x = pack_bf2(u[0], u[1]); pu.y = pack_bf2(u[2], u[3]); pu.z = pack_bf2(u[4], u[5]); pu.w = pack_bf2(u[6], u[7]);
      *reinterpret_cast<uint4*>(blk + (I * TL + i) * 2 * b + J * TL + c) = pu;
      if (I != J) {
        pv.x = pack_bf2(v[0], v[1]); pv.y = pack_bf2(v[2], v[3]); pv.z = pack_bf2(v[4], v[5]); pv.w = pack_bf2(v[6], v[7]);
        *reinterpret_cast<uint4*>(blk + (J * TL + i) * 2 * b + I * TL + c) = pv;
      }
    }
    __syncthreads();
  }
}

// G = 2 (Q + Q2 + Q3) + Q4 + I  (cnp.py:113-115 operation order), 8 columns per thread
__global__ void __launch_bounds__(256) combine_fwd_kernel(int64_t nb, int64_t b, const __nv_bfloat16* __restrict__ qq2,
                                                          const __nv_bfloat16* __restrict__ q34,
                                                          __nv_bfloat16* __restrict__ g16, float* __restrict__ g32) {
  const int64_t nv = nb * b * (b / 8);
  const int64_t cv = b / 8;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nv;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = e / cv;            // s * b + i
    const int c = static_cast<int>(e % cv) * 8;
    const int i = static_cast<int>(row % b);
    const int64_t src = row * 2 * b + c;
    float q[8], q2[8], q3[8], q4[8], v[8];
    unpack_bf8(*reinterpret_cast<const uint4*>(qq2 + src), q);
    unpack_bf8(*reinterpret_cast<const uint4*>(qq2 + src + b), q2);
    unpack_bf8(*reinterpret_cast<const uint4*>(q34 + src), q3);
    unpack_bf8(*reinterpret_cast<const uint4*>(q34 + src + b), q4);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = 2.f * ((q[k] + q2[k]) + q3[k]) + q4[k];
      if (c + k == i) v[k] += 1.f;
    }
    if (g16) *reinterpret_cast<uint4*>(g16 + row * b + c) = pack_bf8(v);
    if (g32) {
      float4* d = reinterpret_cast<float4*>(g32 + row * b + c);
      d[0] = make_float4(v[0], v[1], v[2], v[3]);
      d[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// fp32 -> bf16, 8 per thread
__global__ void __launch_bounds__(256) to_bf16_f32_kernel(int64_t total, const float* __restrict__ x,
                                                          __nv_bfloat16* __restrict__ y) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total / 8;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(x)[2 * e], c = reinterpret_cast<const float4*>(x)[2 * e + 1];
    const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    reinterpret_cast<uint4*>(y)[e] = pack_bf8(v);
  }
}

// in place over n2 (becomes dQ's base): base = 2 (N1 + N2); also
// N2 (bf16), R = 2 N1 + N2 (bf16), P = 2 Q + Q^2 (bf16); 8 columns per thread
__global__ void __launch_bounds__(256) bwd_prep_kernel(int64_t nb, int64_t b, const float* __restrict__ dg,
                                                       float* __restrict__ n2_dq, const __nv_bfloat16* __restrict__ qq2,
                                                       __nv_bfloat16* __restrict__ n2b, __nv_bfloat16* __restrict__ rm,
                                                       __nv_bfloat16* __restrict__ pm) {
  const int64_t nv = nb * b * (b / 8);
  const int64_t cv = b / 8;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nv;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = e / cv;
    const int c = static_cast<int>(e % cv) * 8;
    const int64_t o = row * b + c, src = row * 2 * b + c;
    const float4* n1p = reinterpret_cast<const float4*>(dg + o);
    float4* n2p = reinterpret_cast<float4*>(n2_dq + o);
    const float4 a0 = n1p[0], a1 = n1p[1], b0 = n2p[0], b1 = n2p[1];
    const float n1[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float n2[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float q[8], q2[8], base[8], r[8], p[8];
    unpack_bf8(*reinterpret_cast<const uint4*>(qq2 + src), q);
    unpack_bf8(*reinterpret_cast<const uint4*>(qq2 + src + b), q2);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      base[k] = 2.f * (n1[k] + n2[k]);
      r[k] = 2.f * n1[k] + n2[k];
      p[k] = 2.f * q[k] + q2[k];
    }
    n2p[0] = make_float4(base[0], base[1], base[2], base[3]);
    n2p[1] = make_float4(base[4], base[5], base[6], base[7]);
    *reinterpret_cast<uint4*>(n2b + o) = pack_bf8(n2);
    *reinterpret_cast<uint4*>(rm + o) = pack_bf8(r);
    *reinterpret_cast<uint4*>(pm + o) = pack_bf8(p);
  }
}

// packed grad g_ij = dQ_ij - dQ_ji (cnp.py:81-86) over 64 x 64 tile pairs
__global__ void __launch_bounds__(256) pack_dq_kernel(int64_t nb, int64_t b, const float* __restrict__ dq,
                                                      float* __restrict__ g, int accumulate) {
  __shared__ float lo[TL][TL + 1];  // dQ[J-rows, I-cols]
  const int nt = static_cast<int>(b / TL), npair = nt * (nt + 1) / 2;
  const int64_t pairs = b * (b - 1) / 2;
  const int tx = threadIdx.x % TL, ty = threadIdx.x / TL;
  for (int64_t w = blockIdx.x; w < nb * npair; w += gridDim.x) {
    const int64_t s = w / npair;
    int I, J;
    tile_pair(static_cast<int>(w % npair), nt, I, J);
    const float* blk = dq + s * b * b;
    for (int i = ty; i < TL; i += 4) lo[i][tx] = blk[(J * TL + i) * b + I * TL + tx];
    __syncthreads();
    float* gk = g + s * pairs;
    for (int i = ty; i < TL; i += 4) {
      const int64_t gi = I * TL + i, gj = J * TL + tx;
      if (gj > gi) {
        const float v = blk[gi * b + gj] - lo[tx][i];
        float* dst = gk + pidx(gi, gj, b);
        *dst = accumulate ? *dst + v : v;
      }
    }
    __syncthreads();
  }
}

unsigned tile_grid(int64_t nb, int64_t b) {
  const int64_t nt = b / TL, work = nb * nt * (nt + 1) / 2;
  return static_cast<unsigned>(work < 148 * 16 ? work : 148 * 16);
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

// Stacks are processed in chunks of at most kChunk blocks, so the scratch
// stays bounded (Llama-8B has 11,008 blocks of 256: the whole-stack backward
// scratch would be 8.7 GB) while every launch still covers >= 1024 blocks.
constexpr int64_t kChunk = 1024;

size_t poetx_cnp_tc_workspace_bytes(int64_t nb, int64_t b) {
  if (nb > kChunk) nb = kChunk;
  const size_t blk = static_cast<size_t>(nb * b * b);
  // fwd: Q34 [nb,b,2b] bf16 ; bwd: N1 bf16, N2/dQ fp32, N2 bf16, R bf16, P bf16
  size_t fwd = align_up(blk * 4);
  size_t bwd = align_up(blk * 2) * 4 + align_up(blk * 4);
  return (fwd > bwd ? fwd : bwd) + 4096;
}

static int cnp_forward_tc_chunk(int64_t nb, int64_t b, const float* packed, void* qq2, void* g_bf16,
                                float* g_f32, void* ws, size_t ws_bytes, void* stream);
static int cnp_backward_tc_chunk(int64_t nb, int64_t b, const void* qq2, const float* dg, float* dpacked,
                                 int accumulate, void* ws, size_t ws_bytes, void* stream);

int poetx_cnp_forward_tc(int64_t nb, int64_t b, const float* packed, void* qq2, void* g_bf16,
                         float* g_f32, void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check(nb, b));
  POETX_REQUIRE(packed && qq2 && (g_bf16 || g_f32), POETX_ESHAPE, "cnp_forward_tc: null operand");
  const int64_t pairs = b * (b - 1) / 2;
  for (int64_t o = 0; o < nb; o += kChunk) {
    const int64_t n = nb - o < kChunk ? nb - o : kChunk;
    POETX_TRY(cnp_forward_tc_chunk(n, b, packed + o * pairs, static_cast<__nv_bfloat16*>(qq2) + o * b * 2 * b,
                                   g_bf16 ? static_cast<__nv_bfloat16*>(g_bf16) + o * b * b : nullptr,
                                   g_f32 ? g_f32 + o * b * b : nullptr, ws, ws_bytes, stream));
  }
  return POETX_OK;
}

int poetx_cnp_backward_tc(int64_t nb, int64_t b, const void* qq2, const float* dg, float* dpacked,
                          int accumulate, void* ws, size_t ws_bytes, void* stream) {
  POETX_TRY(check(nb, b));
  POETX_REQUIRE(qq2 && dg && dpacked, POETX_ESHAPE, "cnp_backward_tc: null operand");
  const int64_t pairs = b * (b - 1) / 2;
  for (int64_t o = 0; o < nb; o += kChunk) {
    const int64_t n = nb - o < kChunk ? nb - o : kChunk;
    POETX_TRY(cnp_backward_tc_chunk(n, b, static_cast<const __nv_bfloat16*>(qq2) + o * b * 2 * b, dg + o * b * b,
                                    dpacked + o * pairs, accumulate, ws, ws_bytes, stream));
  }
  return POETX_OK;
}

static int cnp_forward_tc_chunk(int64_t nb, int64_t b, const float* packed, void* qq2, void* g_bf16,
                                float* g_f32, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = as_stream(stream);
  Workspace w(ws, ws_bytes);
  auto* q34 = w.take<__nv_bfloat16>(static_cast<size_t>(nb * b * 2 * b));
  POETX_REQUIRE(q34, POETX_ESHAPE, "cnp_forward_tc: workspace too small");
  auto* QQ2 = static_cast<__nv_bfloat16*>(qq2);
  const int64_t total = nb * b * b;
  unpack_q_kernel<<<tile_grid(nb, b), 256, 0, st>>>(nb, b, packed, QQ2);
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
  combine_fwd_kernel<<<grid_for(total / 8, 256), 256, 0, st>>>(nb, b, QQ2, q34,
                                                           static_cast<__nv_bfloat16*>(g_bf16), g_f32);
  POETX_LAUNCHED("cnp_combine_tc");
  return POETX_OK;
}

static int cnp_backward_tc_chunk(int64_t nb, int64_t b, const void* qq2, const float* dg, float* dpacked,
                                 int accumulate, void* ws, size_t ws_bytes, void* stream) {
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
  to_bf16_f32_kernel<<<grid_for(total / 8, 256), 256, 0, st>>>(total, dg, n1b);
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
  bwd_prep_kernel<<<grid_for(total / 8, 256), 256, 0, st>>>(nb, b, dg, dq, QQ2, n2b, rm, pm);
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
  pack_dq_kernel<<<tile_grid(nb, b), 256, 0, st>>>(nb, b, dq, dpacked, accumulate);
  POETX_LAUNCHED("cnp_pack_tc");
  return POETX_OK;
}

}  // extern "C"
