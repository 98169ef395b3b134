/*
 * poetx_b200.h -- C ABI of the B200-native POET-X hot path.
 *
 * The reference (/root/reference/pkg/src/poetx) is a pure-Python package
 * with no FFI; its "plugin/operator API" for this path is the set of Python
 * functions cited beside each entry point below.  The Python package
 * paper_2603_05500_b200 mirrors those functions one-to-one and reaches the
 * GPU only through this ABI (ctypes).  Any other host
 * (C, C++, Rust, Go via cgo) can bind the same symbols.
 *
 * Conventions
 *   - every pointer named d_* or passed as `void*` data is DEVICE memory
 *     unless stated otherwise; matrices are row-major, contiguous;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *     all device work is stream-ordered, nothing synchronises the host;
 *   - return value: POETX_OK (0) or a positive POETX_E* class code;
 *     poetx_last_error() returns the thread-local message.  The Python
 *     wrapper maps codes to the reference's exception classes
 *     (errors.py:9-42: ShapeError, ConfigError, StateError, NumericsError);
 *   - the library never allocates persistent device memory; callers pass
 *     workspaces sized by the *_workspace_bytes queries.
 */
#ifndef POETX_B200_H
#define POETX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POETX_ABI_VERSION 3

/* element types */
enum { POETX_F32 = 0, POETX_F64 = 1, POETX_BF16 = 2 };
/* status codes (errors.py:9-42) */
enum {
  POETX_OK = 0,
  POETX_ESHAPE = 1,    /* ShapeError   */
  POETX_ECONFIG = 2,   /* ConfigError  */
  POETX_ESTATE = 3,    /* StateError   */
  POETX_ENUMERICS = 4, /* NumericsError */
  POETX_ECUDA = 5      /* CUDA runtime / launch failure */
};
/* layer variants (layer.py:68) */
enum { POETX_FAST = 0, POETX_MEM = 1 };
/* layer boundary flags: let the caller own a permutation so it can be fused
 * into a neighbouring kernel (norm, RoPE, SwiGLU, residual add).  Semantics
 * are unchanged: u = x[:, pi_in], z = v[:, pi_out^-1] (permute.py:95-110). */
enum {
  POETX_IN_GATHERED = 1,     /* x passed is already u = x[:, pi_in] */
  POETX_OUT_UNSCATTERED = 2, /* forward writes v; caller applies z = v[:, pi_out^-1] */
  POETX_DZ_GATHERED = 4,     /* dz passed is already dv = dz[:, pi_out] */
  POETX_DX_UNSCATTERED = 8   /* backward writes du; caller applies dx = du[:, pi_in^-1] */
};

const char* poetx_last_error(void);
int poetx_abi_version(void);
/* number of device kernels this library has launched in this process */
uint64_t poetx_launch_count(void);
/* 1 if the tcgen05/TMA GEMM path is compiled in and enabled */
int poetx_tc_enabled(void);
void poetx_set_tc_enabled(int on);
/* 1 if large single-group BF16 products (mm2, adjoint) run on the CTA-pair
 * (cta_group::2, 256 x 256 tile) kernel; 0 selects the single-CTA kernel */
int poetx_gemm_pair_enabled(void);
void poetx_set_gemm_pair_enabled(int on);
/* A sub-tiles per CTA of the pair GEMM: 0 = by shape (512 x 256 pair tiles
 * for single products with M >= 512), 1 = 256 x 256, 2 = 512 x 256 (A/B) */
void poetx_set_gemm_pair_ms(int ms);
/* device timing hooks: while enabled, tensor-core kernel launches are
 * bracketed by CUDA events on their stream; query sums durations (ms),
 * launch count and algorithmic FLOPs per kernel name ("tc_gemm", ...). */
void poetx_prof_enable(int on);
void poetx_prof_reset(void);
int poetx_prof_query(const char* name, double* total_ms, int64_t* count, double* flops);
/* FP32 CUDA-core peak probe: `ctas` x 256 threads, 8 independent FFMA chains
 * of `iters` each; *flops = FLOP per launch (time it with events on stream). */
int poetx_ffma_probe(int64_t iters, int64_t ctas, float* sink, double* flops, void* stream);

/* ---------------------------------------------------------------- H1 RNG --
 * numpy Generator(Philox) state (the reference draws permutations through
 * numpy: linalg.py:264-291 Rng, permute.py:79-83 sample_permutation).
 * HOST memory.  Bit-exact with numpy 2.x: counter pre-increment, 4-word
 * buffer, low-then-high uint32 halves, masked-rejection bounded ints,
 * Fisher-Yates for i = n-1 .. 1.                                            */
typedef struct {
  uint64_t counter[4];
  uint64_t key[2];
  uint64_t buffer[4];
  int64_t buffer_pos;
  int64_t has_uint32;
  uint64_t uinteger;
} poetx_philox_state;

/* fresh stream: Rng(seed, stream) (linalg.py:276-279) */
int poetx_philox_seed(poetx_philox_state* st, uint64_t seed, uint64_t stream);
/* Rng.permutation(n) -> forward map and its inverse (host int32[n] each;
 * inv may be NULL) (linalg.py:290-291, permute.py:65-76) */
int poetx_philox_permutation(poetx_philox_state* st, int64_t n, int32_t* fwd, int32_t* inv);

/* ------------------------------------------------------------------ CNP --
 * cnp.py.  dtype in {F32, F64}: Q, G, caches and grads in that type.
 * dtype BF16 is not a CNP dtype (parameters stay fp32 master); use F32 and
 * request a bf16 copy of G through g_bf16.                                 */

/* skew_from_packed (cnp.py:71-78): q[nb,b,b] from packed[nb, b(b-1)/2] */
int poetx_skew_from_packed(int dtype, int64_t nb, int64_t b, const void* packed, void* q,
                           void* stream);
/* packed_grad_from_skew_grad (cnp.py:81-86): g_ij = dq_ij - dq_ji;
 * accumulate != 0 adds into g */
int poetx_packed_grad_from_skew_grad(int dtype, int64_t nb, int64_t b, const void* dq,
                                     void* g, int accumulate, void* stream);
size_t poetx_cnp_workspace_bytes(int dtype, int64_t nb, int64_t b, int k);
/* cnp_forward (cnp.py:99-125).  Input: q (full skew stack) if q != NULL,
 * else packed params (unpacked in-kernel).  Outputs: g (required),
 * g_bf16 (optional bf16 copy for the tensor-core path), q2 (optional
 * cache of Q^2, k == 3 only). */
int poetx_cnp_forward(int dtype, int64_t nb, int64_t b, int k, const void* q,
                      const void* packed, void* g, void* g_bf16, void* q2, void* ws,
                      size_t ws_bytes, void* stream);
/* cnp_backward (cnp.py:128-158), optionally fused with
 * packed_grad_from_skew_grad (cnp.py:81-86).  q / packed as above;
 * q2 may be NULL (recomputed).  Writes dq (full stack) if dq != NULL and
 * the packed gradient if dpacked != NULL (accumulate != 0 adds). */
int poetx_cnp_backward(int dtype, int64_t nb, int64_t b, int k, const void* q,
                       const void* packed, const void* q2, const void* dg, void* dq,
                       void* dpacked, int accumulate, void* ws, size_t ws_bytes, void* stream);
/* Tensor-core CNP for the BF16 path, k = 3, b in {64, 128, 256}, over a
 * stack of nb blocks (e.g. every block of a model: the packed parameters
 * are one flat buffer).  Forward: packed fp32 [nb, b(b-1)/2] ->
 * qq2 = [Q | Q^2] bf16 [nb, b, 2b] (the backward's cache) and
 * G = I + 2(Q+Q^2+Q^3) + Q^4 as bf16 and/or fp32 [nb, b, b]
 * (cnp.py:99-116).  Backward: dG fp32 [nb, b, b] -> packed fp32 gradient
 * via dQ = 2(N1+N2) + (2Q+Q^2)^T N2 + (2N1+N2)(Q^2)^T, N2 = -(N1 Q + Q N1)
 * (cnp.py:128-145 regrouped) and g_ij = dQ_ij - dQ_ji. */
/* Fused tensor-core CNP (k = 3, bf16 operands, fp32 accumulation in TMEM),
 * one kernel per direction, b in {128, 256} (cnp.py:71-158 + 81-86):
 * forward packed fp32 [nb, b(b-1)/2] -> G bf16 [nb, b, b] (and/or fp32);
 * backward packed + dG fp32 [nb, b, b] -> packed gradient (+= if accumulate).
 * No cache between the two (the backward recomputes Q^2 on chip); no
 * workspace.  poetx_cnp_fused_supported(b) says whether b is handled. */
int poetx_cnp_fused_supported(int64_t b);
int poetx_cnp_forward_fused(int64_t nb, int64_t b, const float* packed, void* g_bf16, float* g_f32, void* stream);
int poetx_cnp_backward_fused(int64_t nb, int64_t b, const float* packed, const float* dg, float* dpacked,
                             int accumulate, void* stream);
size_t poetx_cnp_tc_workspace_bytes(int64_t nb, int64_t b);
int poetx_cnp_forward_tc(int64_t nb, int64_t b, const float* packed, void* qq2, void* g_bf16,
                         float* g_f32, void* ws, size_t ws_bytes, void* stream);
int poetx_cnp_backward_tc(int64_t nb, int64_t b, const void* qq2, const float* dg, float* dpacked,
                          int accumulate, void* ws, size_t ws_bytes, void* stream);
/* cayley-free orthogonality audit ||G^T G - I||_F over the stack
 * (blockdiag.py:134-138).  out: DEVICE double[1]. */
int poetx_orthogonality_error(int dtype, int64_t nb, int64_t b, const void* g, double* out,
                              void* ws, size_t ws_bytes, void* stream);

/* ----------------------------------------------------- permutations -----
 * permute.py.  These are exact data movement in any dtype.                */
/* y[i, j] = x[i, idx[j]]   (permute_cols / permute_features, permute.py:95-110:
 * 'forward' passes idx = pi.inverse, 'inverse' passes idx = pi.forward) */
int poetx_permute_cols(int dtype, int64_t rows, int64_t cols, const int32_t* idx,
                       const void* x, void* y, void* stream);
/* y[i, :] = x[idx[i], :]   (permute_rows, permute.py:86-92) */
int poetx_permute_rows(int dtype, int64_t rows, int64_t cols, const int32_t* idx,
                       const void* x, void* y, void* stream);
/* y[i, j] = x[ridx[i], cidx[j]]  (premerge_weight, permute.py:113-125;
 * also the composite re-permutation of merge_and_reinit) */
int poetx_gather2d(int dtype, int64_t rows, int64_t cols, const int32_t* ridx,
                   const int32_t* cidx, const void* x, void* y, void* stream);

/* ------------------------------------------------------- block-diagonal --
 * blockdiag.py.  g is (nb, b, b) in dtype (BF16 activations take a BF16 g). */
/* apply_to_features (blockdiag.py:58-73): y_s = x_s g[s] (or g[s]^T) */
int poetx_apply_to_features(int dtype, int64_t T, int64_t nb, int64_t b, const void* g,
                            int transpose, const void* x, void* y, void* stream);
/* apply_to_weight_rows (blockdiag.py:76-90): y_s = g[s] w_s (or g[s]^T w_s) */
int poetx_apply_to_weight_rows(int dtype, int64_t nb, int64_t b, int64_t cols, const void* g,
                               int transpose, const void* w, void* y, void* stream);
size_t poetx_segmented_outer_workspace_bytes(int dtype, int64_t T, int64_t nb, int64_t b);
/* segmented_outer (blockdiag.py:100-121): out[s] = sum_t x_s^T y_s.
 * out is F64 for F64 inputs and F32 otherwise (BF16 inputs accumulate in
 * fp32).  Deterministic split-T reduction.  accumulate != 0 adds. */
int poetx_segmented_outer(int dtype, int64_t T, int64_t nb, int64_t b, const void* x,
                          const void* y, void* out, int accumulate, void* ws, size_t ws_bytes,
                          void* stream);

/* ---------------------------------------------------------------- GEMM --
 * C[M,N] (+)= op(A)[M,K] op(B)[K,N]; lda/ldb/ldc are row strides of the
 * stored (untransposed) arrays.  linalg.matmul / matmul_abt
 * (linalg.py:42-83) are (transB = 0 / 1).  BF16 inputs accumulate in fp32
 * and store BF16; with tc enabled BF16 shapes that tile evenly run on the
 * tcgen05/TMA kernel. */
int poetx_matmul(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                 int transA, const void* B, int64_t ldb, int transB, void* C, int64_t ldc,
                 int accumulate, void* stream);
/* POET-XQ product with the frozen weight's int8 codes dequantized inside the
 * GEMM producer (layer.py:188-210 with quant.py's per-row scales): BF16
 * C[M,N] = A[M,K] . W, W = codes[K,N] * scales[k] (transB = 0) or
 * W = (codes[N,K] * scales[n])^T (transB = 1); each element rounded to bf16
 * once, exactly as poetx_dequantize_rows, so the result is bit-identical to
 * dequantize + poetx_matmul.  CTA-pair tcgen05 kernel only (N % 256 == 0,
 * 16-byte aligned pitches), else POETX_ESHAPE. */
int poetx_matmul_q8(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const int8_t* codes, int64_t ldb,
                    int transB, const float* scales, void* C, int64_t ldc, void* stream);

/* ---------------------------------------------------------------- layer --
 * PoetLinearLayer forward/backward (layer.py:214-256) as one call each.  */
typedef struct {
  int dtype;        /* activation / frozen-weight type: F32, F64 or BF16 */
  int variant;      /* POETX_FAST or POETX_MEM */
  int neumann_k;
  int64_t m, n, b;  /* in-features, out-features, block size */
  const int32_t* perm_in_fwd;  /* device int32[m] */
  const int32_t* perm_in_inv;
  const int32_t* perm_out_fwd; /* device int32[n] */
  const int32_t* perm_out_inv;
  const void* premerged;       /* device [m, n] = W[pi_in(i), pi_out(j)] */
  /* POET-XQ (mem variant only, quant.py): when pm_codes != NULL the frozen
   * weight is int8 codes [m, n] of the premerged matrix with per-row scales
   * [m] (F64 for F64 layers, else F32) and premerged is ignored.  BF16
   * layers at b = 256 feed the codes straight into the pair GEMM's producer
   * (dequantized on chip); other shapes dequantize into the call's workspace
   * right before the product. */
  const int8_t* pm_codes;
  const void* pm_scales;
  /* BF16 layers: nonzero -> reassociated products, the block factors folded
   * into the frozen weight (bd(G_R) PM, PM bd(G_P)) -- fewer bytes
   * when T is large against n*b; zero -> factors applied to the activations. */
  int fold_weight;
  /* optional caller-owned stream (cudaStream_t) for the backward's two
   * segmented outer products, forked and joined with per-call events; NULL:
   * everything on the call's stream.  Must differ from the call's stream. */
  void* side_stream;
} poetx_layer_desc;

/* factor state produced by poetx_layer_factors and consumed by fwd/bwd.
 * Parameter/factor type: F64 for F64 layers, else F32 (fp32 master). */
typedef struct {
  const void* packed_r;  /* [m/b, b(b-1)/2] */
  const void* packed_p;  /* [n/b, b(b-1)/2] */
  void* g_r;             /* [m/b, b, b] param type */
  void* g_p;
  void* g_r_lowp;        /* BF16 copies (BF16 layers only, else NULL) */
  void* g_p_lowp;
  void* q2_r;            /* Q^2 caches (k == 3), may be NULL.  A BF16 layer with
                          * k == 3, b in {128, 256} and BOTH caches NULL runs
                          * its CNP as the fused tensor-core kernels
                          * (poetx_cnp_forward_fused / _backward_fused);
                          * supplying the caches selects the fp32 CUDA-core
                          * CNP (the merge uses it for accuracy). */
  void* q2_p;
  /* optional precomputed weight folds of a BF16 layer (else built per call):
   * w_in_fold = bd(G_R) PM, w_out_fold = PM bd(G_P), both [m, n] bf16 --
   * for a POET-XQ layer with b = 256 and m % 256 == 0, w_out_fold is stored
   * transposed ([n, m]), as poetx_layer_weight_fold(which = 1) writes it */
  const void* w_in_fold;
  const void* w_out_fold;
} poetx_layer_factors_t;

size_t poetx_layer_workspace_bytes(const poetx_layer_desc* d, int64_t T);
/* BF16 weight folds: which = 0 -> out = bd(G_R) PM, 1 -> out =
 * PM bd(G_P), from the factors' bf16 G; out is [m, n] bf16.  POET-XQ bases:
 * the int8 codes are dequantized inside the GEMM producer where the pair
 * kernel takes them (b = 256), and which = 1 then writes (PM bd(G_P))^T,
 * [n, m], the layout the layer backward reads.  ws >= poetx_layer_workspace_bytes(d, 0). */
int poetx_layer_weight_fold(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int which, void* out,
                            void* ws, size_t ws_bytes, void* stream);
int poetx_layer_factors(const poetx_layer_desc* d, poetx_layer_factors_t* f, void* ws,
                        size_t ws_bytes, void* stream);
/* z[T,n] = layer(x[T,m]); saved_t[T,n] written when non-NULL (fast). */
int poetx_layer_forward(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                        const void* x, void* z, void* saved_t, void* ws, size_t ws_bytes,
                        void* stream);
/* forward with boundary flags (POETX_IN_GATHERED, POETX_OUT_UNSCATTERED) */
int poetx_layer_forward_ex(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                           const void* x, void* z, void* saved_t, int flags, void* ws,
                           size_t ws_bytes, void* stream);
/* grads: dx[T,m] (may be NULL), packed grads (param type; accumulate != 0
 * adds into them).  saved_t NULL => recompute (mem variant). */
int poetx_layer_backward(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                         const void* x, const void* dz, const void* saved_t, void* dx,
                         void* dpacked_r, void* dpacked_p, int accumulate, void* ws,
                         size_t ws_bytes, void* stream);
/* Same chain, but instead of running the CNP backward per layer it leaves
 * the block-factor cotangents dG_R [m/b,b,b], dG_P [n/b,b,b] (fp32; F64 for
 * F64 layers) in caller buffers (accumulate != 0 adds) so one batched
 * poetx_cnp_backward_tc can serve every layer of a model.  flags:
 * POETX_IN_GATHERED (x is u), POETX_DZ_GATHERED, POETX_DX_UNSCATTERED. */
int poetx_layer_backward_dg(const poetx_layer_desc* d, const poetx_layer_factors_t* f, int64_t T,
                            const void* x, const void* dz, const void* saved_t, void* dx,
                            void* dg_r, void* dg_p, int accumulate, int flags, void* ws,
                            size_t ws_bytes, void* stream);
/* merge_and_reinit numerics (layer.py:260-314): new premerged
 * PM'[i,j] = M[inv_in(new_in(i)), inv_out(new_out(j))] with
 * M = blockdiag(G_R) PM blockdiag(G_P) computed in fp32/fp64 from the
 * given factors; optional W_out = Psi^T M Psi (materialize_weight).
 * premerged_out (codes_out / scales_out) may be the layer's own buffers:
 * the old weight is read only before the final re-permutation gather. */
size_t poetx_merge_workspace_bytes(const poetx_layer_desc* d);
/* Tensor-core merge product (kernel K9; layer.py:260-271, blockdiag.py:76-97):
 * out = blockdiag(G_R) PM blockdiag(G_P) for fp32 factors G_R [m/b, b, b],
 * G_P [n/b, b, b] and a bf16 premerged PM [m, ldp] -- or int8 codes [m, ldp]
 * with per-row fp32 scales (POET-XQ, PM = codes * scales[row]) when pm_bf16
 * is NULL.  Factors are split on chip into bf16 hi + lo (fp32 accumulation
 * in TMEM; only the lo*lo term is dropped).  out is bf16 or fp32 [m, ldo].
 * b in {128, 256} (poetx_merge_tc_supported); no workspace.  Used by
 * poetx_layer_merge / _merge_quant for BF16 layers. */
int poetx_merge_tc_supported(int64_t b);
int poetx_merge_tc(int64_t m, int64_t n, int64_t b, const float* g_r, const float* g_p, const void* pm_bf16,
                   const int8_t* pm_codes, const float* pm_scales, int64_t ldp, void* out, int out_dtype,
                   int64_t ldo, void* stream);
int poetx_layer_merge(const poetx_layer_desc* d, const void* g_r, const void* g_p,
                      const int32_t* new_in_fwd, const int32_t* new_out_fwd,
                      void* premerged_out, void* w_out, void* ws, size_t ws_bytes,
                      void* stream);

/* POET-XQ merge (layer.py:279-314 with a quantized base): the transformed
 * base is requantized per row (bit-exact rule of quant.py:41-48) and the
 * new premerged codes/scales are gathered in the quantized domain. */
int poetx_layer_merge_quant(const poetx_layer_desc* d, const void* g_r, const void* g_p,
                            const int32_t* new_in_fwd, const int32_t* new_out_fwd, int8_t* codes_out,
                            void* scales_out, void* w_out, void* ws, size_t ws_bytes, void* stream);

/* ----------------------------------------------------------------- quant --
 * Per-row symmetric int8 (quant.py:22-74).  dtype = float type of w / out;
 * scales are F64 for F64, else F32.  Round half to even, codes in
 * [-127, 127], all-zero rows get scale 1.0 -- bit-exact with the reference. */
int poetx_quantize_rows(int dtype, int64_t rows, int64_t cols, const void* w, int8_t* codes, void* scales,
                        void* stream);
/* out[i, j] = codes[ri(i), ci(j)] * scales[ri(i)] for an output [rows, cols];
 * codes rows are src_cols long; row_idx/col_idx may be NULL */
int poetx_dequantize_rows(int dtype, int64_t rows, int64_t cols, int64_t src_cols, const int8_t* codes,
                          const void* scales, const int32_t* row_idx, const int32_t* col_idx, void* out,
                          void* stream);
/* quantized-domain gather into [rows, cols] (exact: commutes with dequantization) */
int poetx_quant_gather(int dtype, int64_t rows, int64_t cols, int64_t src_cols, const int32_t* row_idx,
                       const int32_t* col_idx, const int8_t* codes, const void* scales, int8_t* codes_out,
                       void* scales_out, void* stream);

/* ----------------------------------------------------------- loss head --
 * cross_entropy_fwd: per-row loss over bf16 logits [T, V] (V % 8 == 0) with
 * row max / sum-exp kept for the backward; cross_entropy_bwd: bf16
 * dlogits = (softmax - onehot) * (*dloss) * scale.  A target outside
 * [0, V) (e.g. an ignore_index) is rejected: NaN loss row, zero grad row. */
int poetx_cross_entropy_fwd(int64_t T, int64_t V, const void* logits, const int64_t* targets, float* loss_rows,
                            float* row_max, float* row_sumexp, void* stream);
int poetx_cross_entropy_bwd(int64_t T, int64_t V, const void* logits, const int64_t* targets, const float* row_max,
                            const float* row_sumexp, const float* dloss, float scale, void* dlogits, void* stream);

/* ------------------------------------------------------------ embedding --
 * The trainer's token embedding (model plumbing): out[t] = bf16(table[tok[t]])
 * (fp32 table [V, d]); backward: dtable[v] += sum_{tok[t] = v} dh[t] over the
 * tokens sorted stably by id (sorted_tokens, order = the sort's permutation),
 * one warp per id in ascending position order -- deterministic, no atomics.
 * Ids outside [0, V) never address the table: the forward writes a NaN row
 * and the backward skips them. */
int poetx_embedding_fwd(int64_t T, int64_t V, int64_t d, const int64_t* tokens, const float* table, void* out,
                        void* stream);
int poetx_embedding_bwd(int64_t T, int64_t V, int64_t d, const int64_t* sorted_tokens, const int64_t* order,
                        const void* dh, float* dtable, void* stream);

/* ---------------------------------------------------- singular values --
 * svd_singular_values (linalg.py:166-218): one-sided Jacobi in float64,
 * same rotation and stopping rule (tol relative to sqrt(alpha beta), stop
 * after a rotation-free sweep), round-robin pair order, one CTA per matrix.
 * a: batch row-major [rows, cols] float64; sv: batch x min(rows, cols),
 * descending.  residual / sweeps (optional, per matrix): worst relative
 * off-diagonal of the last sweep (0 when converged) and the sweeps used, -1
 * when max_sweeps ran out (the caller raises ConvergenceError).
 * min(rows, cols) <= 4096. */
size_t poetx_singular_values_workspace_bytes(int64_t batch, int64_t rows, int64_t cols);
int poetx_singular_values(int64_t batch, int64_t rows, int64_t cols, const double* a, double* sv, double tol,
                          int max_sweeps, double* residual, int* sweeps, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------ attention backward --
 * Causal softmax attention backward, bf16, token-major [B*S, H*hd] tensors
 * (row pitch H*hd), natural-log logsumexp lse [B, H, S] from the forward
 * (cuDNN's).  dq/dk/dv are written (not accumulated).  Supported shape: S =
 * 256, hd = 64 (the Llama-60M/350M/1B blocks); anything else returns
 * POETX_ECONFIG.  Model plumbing, not a reference interface. */
int poetx_attention_bwd(int64_t B, int64_t S, int64_t H, int64_t hd, const void* q, const void* k, const void* v,
                        const void* o, const void* dout, const float* lse, void* dq, void* dk, void* dv,
                        void* stream);

/* ------------------------------------------------ fused neighbour kernels --
 * BF16 row-staged kernels that apply the layer permutations inside the
 * elementwise ops a decoder block needs anyway (used with the
 * POETX_IN_GATHERED / POETX_OUT_UNSCATTERED layer flags).  All index
 * arrays are DEVICE int32; rows are [T, dim] row-major, dim % 8 == 0.   */
/* y = rmsnorm(x) * w (fp32 math), out[k] = y[:, idx[k]] for k < K <= 3;
 * rstd[T] (fp32) saved for the backward */
int poetx_rmsnorm_gather(int64_t T, int64_t d, const void* x, const float* w, float eps, int K,
                         const int32_t* const* idx, void* const* out, float* rstd, void* stream);
size_t poetx_rmsnorm_gather_bwd_workspace_bytes(int64_t T, int64_t d);
/* dy = sum_k du[k][:, inv[k]]; dx = RMSNorm backward (+ dres, the residual
 * stream's own gradient, when non-NULL); dw (+)= sum_t dy x rstd
 * (deterministic per-CTA partials) */
int poetx_rmsnorm_gather_bwd(int64_t T, int64_t d, const void* x, const float* w, const float* rstd,
                             int K, const int32_t* const* inv, const void* const* du,
                             const void* dres, void* dx, float* dw, int accumulate_dw, void* ws,
                             size_t ws_bytes, void* stream);
/* out[:, j] = silu(vg[:, cg[j]]) * vu[:, cu[j]] */
int poetx_swiglu_gather(int64_t T, int64_t f, const void* vg, const void* vu, const int32_t* cg,
                        const int32_t* cu, void* out, void* stream);
/* dvg[:, j] = du[:, A[j]] silu'(vg[:, j]) vu[:, B[j]];  dvu[:, j] = du[:, C[j]] silu(vg[:, D[j]]).
 * The maps of one SwiGLU satisfy C = A o D (C[j] = A[D[j]]); the kernel uses
 * that (dvu formed in gate order, then gathered through D) and does not read C. */
int poetx_swiglu_gather_bwd(int64_t T, int64_t f, const void* vg, const void* vu, const void* du,
                            const int32_t* A, const int32_t* B, const int32_t* C, const int32_t* D,
                            void* dvg, void* dvu, void* stream);
/* the same with 16-bit maps (f <= 65536): half the index bytes through L1 */
int poetx_swiglu_gather16(int64_t T, int64_t f, const void* vg, const void* vu, const uint16_t* cg,
                          const uint16_t* cu, void* out, void* stream);
int poetx_swiglu_gather_bwd16(int64_t T, int64_t f, const void* vg, const void* vu, const void* du,
                              const uint16_t* A, const uint16_t* B, const uint16_t* C, const uint16_t* D,
                              void* dvg, void* dvu, void* stream);
/* out = RoPE(v[:, inv]) per head (pairs c, c + hd/2; position t % S) */
int poetx_rope_scatter(int64_t T, int64_t S, int64_t H, int64_t hd, const void* v,
                       const int32_t* inv, const float* cosb, const float* sinb, void* out,
                       void* stream);
int poetx_rope_scatter_bwd(int64_t T, int64_t S, int64_t H, int64_t hd, const void* dout,
                           const int32_t* fwd, const float* cosb, const float* sinb, void* dv,
                           void* stream);
/* out = h + v[:, inv]  (residual add with the output scatter) */
int poetx_scatter_add(int64_t T, int64_t d, const void* h, const void* v, const int32_t* inv,
                      void* out, void* stream);

/* ------------------------------------------------------------ optimizer --
 * optim.py.  Multi-tensor: host arrays of device pointers.               */
/* sum of squares in float64 over all tensors into DEVICE double out[0]
 * (global_grad_norm, optim.py:77-81, squared); nonfinite (DEVICE int) is
 * set to 1 if any element is inf/nan. */
int poetx_sqnorm(int dtype, int ntensors, const void* const* g, const int64_t* numel,
                 double* out, int* nonfinite, void* ws, size_t ws_bytes, void* stream);
size_t poetx_sqnorm_workspace_bytes(int ntensors, const int64_t* numel);
/* fused clip + AdamW (optim.py:84-94 + 127-148), arithmetic in the param
 * type with the reference's operation order.  If sqnorm != NULL (DEVICE
 * double) and sqrt(*sqnorm) > clip_threshold, grads are first scaled by
 * (type)(clip_threshold / norm) -- written back to g when write_back_grads;
 * a non-finite *sqnorm skips the update (nothing is written).
 * bc1 = 1 - beta1^t, bc2 = 1 - beta2^t computed by the caller in double. */
int poetx_adamw(int dtype, int ntensors, void* const* p, void* const* g, void* const* m,
                void* const* v, const int64_t* numel, double lr, double beta1, double beta2,
                double eps, double weight_decay, double bc1, double bc2, const double* sqnorm,
                double clip_threshold, int write_back_grads, void* stream);

/* same update with the step-dependent scalars read from DEVICE memory
 * dyn = {lr, lr*weight_decay, 1-beta1^t, 1-beta2^t, clip_threshold} (double),
 * so a captured CUDA graph replays every step with fresh values. */
int poetx_adamw_dyn(int dtype, int ntensors, void* const* p, void* const* g, void* const* m,
                    void* const* v, const int64_t* numel, double beta1, double beta2, double eps,
                    const double* dyn, const double* sqnorm, int write_back_grads, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* POETX_B200_H */
