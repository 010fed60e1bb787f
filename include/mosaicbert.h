/* mosaicbert.h — C ABI of the B200 (sm_100a) MosaicBERT data-parallel hot path.
 *
 * Paper: "MosaicBERT: A Bidirectional Encoder Optimized for Fast Pretraining" (arXiv 2312.17482).
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R-numbers = readings listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Pointers marked "device" are CUDA device pointers owned by the caller (allocated by torch in
 *    the Python layer).  The library keeps no device state and allocates nothing: every scratch
 *    buffer is a caller workspace sized by an mb_*_workspace_bytes() query.
 *  - Every device call is ordered on the given stream `s` (a cudaStream_t; NULL = legacy default)
 *    and never synchronises the host.  Results are visible after the stream reaches them.
 *  - bf16 tensors are raw bfloat16 bit patterns (uint16_t), row-major, densely packed unless a
 *    leading dimension is given.  Weights follow nn.Linear: W[out, in].
 *  - Gradients are fp32 and ACCUMULATED (+=): the caller zeroes them once per optimizer step, so
 *    gradient accumulation over micro-steps is free ("float32 for gradient accumulation").
 *  - Host-checkable argument errors return a status immediately and launch nothing.  Data-dependent
 *    errors (mask layout, token-id range, label range) are written to a device status word (meta[2])
 *    that the caller reads at its own sync point.  Launch failures return MB_ERR_CUDA.  Every entry
 *    point that touches the device returns MB_ERR_ARCH (and launches nothing) when the current
 *    device is not sm_100 (B200): the library carries sm_100a SASS only.  No C++ exception crosses
 *    the ABI.
 *  - Calls are reentrant and may run concurrently on different streams (each call uses only the
 *    buffers passed to it); the only global state is a per-device attribute cache (SM count,
 *    architecture) and the instrumentation counters below.
 */
#ifndef MOSAICBERT_H_
#define MOSAICBERT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MB_API __attribute__((visibility("default")))
#else
#define MB_API
#endif

typedef struct CUstream_st* mb_stream_t; /* == cudaStream_t */
typedef uint16_t mb_bf16;                /* raw bfloat16 bits */

typedef enum {
  MB_OK = 0,
  MB_ERR_INVALID_ARG = 1, /* null pointer, negative size                                             */
  MB_ERR_CONFIG = 2,      /* heads<=0, hidden%heads!=0, head_dim not in {32,64},
                             odd fused GLU width, vocab<1, dims not multiples of 8           */
  MB_ERR_SHAPE = 3,       /* nnz > B*L, max_seqlen > 2048, n_masked > nnz                            */
  MB_ERR_MASK_LAYOUT = 4, /* device-reported: a mask row is not a right-padded prefix (R6)    */
  MB_ERR_LABEL_RANGE = 5, /* device-reported: label not in [0, V)                                    */
  MB_ERR_WORKSPACE = 6,   /* workspace smaller than mb_*_workspace_bytes(...)                        */
  MB_ERR_ARCH = 7,        /* device is not sm_100 (B200)                                             */
  MB_ERR_CUDA = 8,        /* CUDA launch / runtime error                                             */
  MB_ERR_TOKEN_RANGE = 9  /* device-reported: a real token's id is not in [0, V) (A3 reads E_tok[id]) */
} mb_status;

MB_API const char* mb_status_string(int status);
/* Library version string and the SASS target it was built for ("sm_100a"). */
MB_API const char* mb_version(void);

/* Instrumentation (host only; not used by the compute path):
 *  mb_launch_count: total kernels this process has launched through the library (monotonic).
 *  mb_probe_set: record caller-created cudaEvent_t pairs around every launch of one kernel site so
 *    that a benchmark can time that kernel inside a real step on the stream it runs on.
 *    site: 0 = off, 1 = GeGLU up-projection GEMM (A8), 2 = attention fwd (A5), 3 = attention bwd
 *    (A10), 4 = LayerNorm fwd (A7).  events: host array of `capacity` cudaEvent_t (pairs
 *    start/end); *count (host int) is incremented per recorded pair.  Not thread-safe. */
MB_API unsigned long long mb_launch_count(void);
MB_API mb_status mb_probe_set(int32_t site, void* events, int32_t capacity, int32_t* count);

/* Model dimensions.  d = hidden/heads (head_dim, 32 or 64).  ln_eps: LayerNorm epsilon (R11).
 * flags: MB_FLAG_DETERMINISTIC makes every gradient reduction of mb_encoder_backward, mb_mlm_loss and
 *   mb_embed_backward bitwise reproducible from run to run: split-K weight-
 *   gradient partials are added split by split in split order (per-tile turnstiles), per-CTA column
 *   partials (LN dgamma/dbeta, bias gradients) are summed in a fixed order by a second pass, the
 *   long-sequence dQ is kept per key tile and summed in key-tile order, and the embedding-table
 *   scatter-add sums the rows of each token id in token order.  The default (0) uses fp32 atomics:
 *   faster, equal up to fp32 reassociation.  The workspace queries take the flag into account. */
enum { MB_FLAG_DETERMINISTIC = 1 };
typedef struct {
  int32_t hidden, heads, intermediate, vocab;
  float ln_eps;
  int32_t flags;
} mb_dims;

/* ---------------------------------------------------------------------------------------------
 * ALiBi slopes (host, pure).  out[h] = (float)2^(-8(h+1)/heads), h = 0..heads-1.
 * P:129 "The slopes m follow a geometric sequence such that for n heads, each head has a ratio of
 * 2^{-8/n}" (reading R3/R27: first term equals the ratio).  out: host float[heads].
 * Errors: heads <= 0 -> MB_ERR_CONFIG; out == NULL -> MB_ERR_INVALID_ARG. */
MB_API mb_status mb_alibi_slopes(int32_t heads, float* host_out);

/* ---------------------------------------------------------------------------------------------
 * A1 — unpad index ("concatenate all the examples from a minibatch into a single sequence of
 * batch size 1").
 *   mask       device int32[B*L], 1 = real token, right-padded rows (R6).
 *   ids        device int32[B*L] token ids, or NULL: if given, every REAL position's id is checked
 *              against [0, vocab) (the embedding gathers E_tok[id]; upstream nn.Embedding
 *              raises on such ids) — a violation sets status MB_ERR_TOKEN_RANGE.
 *   cu_seqlens device int32[B+1] out: [0, cumsum(seqlen)]  (non-decreasing; zero-length rows OK, R5)
 *   indices    device int32[B*L] out (capacity): first nnz entries = ascending flat positions b*L+l
 *              with mask==1 (the flash-attention `unpad_input` convention)
 *   meta       device int32[4] out: {nnz, max_seqlen, status, (unchanged)}; status = MB_OK,
 *              MB_ERR_MASK_LAYOUT if some row is not a prefix of ones (precedence; indices are still
 *              the positions of the ones), else MB_ERR_TOKEN_RANGE for a bad id.
 *   ws         device workspace of mb_unpad_workspace_bytes(B) bytes (per-row counts and status), or
 *              NULL (then a single-CTA kernel does the whole scan: same results, slower at large B).
 * Bit-exact by construction (integer work).  Limits: B <= 65536, L <= 65536.
 * Errors: NULL mask/cu/indices/meta or B, L outside [1, 65536] -> MB_ERR_INVALID_ARG; ids given with
 * vocab < 1 -> MB_ERR_CONFIG; ws_bytes too small -> MB_ERR_WORKSPACE. */
MB_API size_t mb_unpad_workspace_bytes(int32_t B);
MB_API mb_status mb_unpad_index(const int32_t* mask, const int32_t* ids, int32_t vocab, int32_t B, int32_t L,
                                int32_t* cu_seqlens, int32_t* indices, int32_t* meta, void* ws, size_t ws_bytes,
                                mb_stream_t s);

/* MLM selection: among the packed tokens t < meta[0] (device nnz), select those
 * whose padded label labels[indices[t]] != -100.
 *   masked_rows   device int32[capacity] out: packed row ids t (ascending)
 *   masked_labels device int32[capacity] out: their labels
 *   meta          device int32[4] in/out: reads meta[0] (nnz); writes meta[3] = n_masked and sets
 *                 meta[2] = MB_ERR_LABEL_RANGE if a selected label is outside [0, vocab).
 *   count_accum   device fp32 scalar or NULL: += n_masked (the R18 normaliser of an optimizer step is
 *                 this sum over its micro-steps — and over the data-parallel ranks after an allreduce —
 *                 so the loss scale never needs a device->host read).
 *   ws            device workspace of mb_select_workspace_bytes(capacity) bytes, or NULL (single-CTA
 *                 kernel).  Errors: ws_bytes too small -> MB_ERR_WORKSPACE. */
MB_API size_t mb_select_workspace_bytes(int32_t capacity);
MB_API mb_status mb_mlm_select(const int32_t* labels, const int32_t* indices, int32_t capacity, int32_t vocab,
                               int32_t* masked_rows, int32_t* masked_labels, int32_t* meta, float* count_accum,
                               void* ws, size_t ws_bytes, mb_stream_t s);

/* A2 — row gather / scatter between the padded [rows, H] and packed [n, H] layouts.
 *   gather : dst[t,:] = src[idx[t],:]                       (unpad)
 *   scatter: dst[idx[t],:] = src[t,:], all other rows of dst set to exactly 0 (pad)
 * H must be a multiple of 8 (16-byte vectors).  idx device int32[n]. */
MB_API mb_status mb_gather_rows(const mb_bf16* src, const int32_t* idx, int32_t n, int32_t H, mb_bf16* dst,
                         mb_stream_t s);
MB_API mb_status mb_scatter_rows(const mb_bf16* src, const int32_t* idx, int32_t n, int32_t H, int32_t rows,
                          mb_bf16* dst, mb_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * Building blocks (exported so that every kernel can be parity-tested on its own).
 * ------------------------------------------------------------------------------------------- */

/* A7 — bf16 LayerNorm ("we modify LayerNorm modules to run in bfloat16 precision").
 * x, y bf16 [n, H]; gamma, beta bf16 [H]; stats fp32 [n, 2] out = {mean, rstd}.
 * y = (x - mean) * rstd * gamma + beta, stats and arithmetic in fp32, y rounded once (R12). */
MB_API mb_status mb_layernorm_forward(const mb_bf16* x, const mb_bf16* gamma, const mb_bf16* beta, int32_t n,
                               int32_t H, float eps, mb_bf16* y, float* stats, mb_stream_t s);
/* LN backward: dx = rstd (g - mean(g) - xhat mean(g xhat)), g = dy*gamma; accumulates (+=) fp32
 * dgamma = sum dy*xhat, dbeta = sum dy, and (if dsum != NULL) dsum = sum dx — the bias gradient of
 * the linear layer that produced x.  If gelu_pre != NULL the result is multiplied by
 * GeLU'(gelu_pre) (the MLM-transform backward, A11).  dx may alias dy. */
MB_API mb_status mb_layernorm_backward(const mb_bf16* dy, const mb_bf16* x, const float* stats, const mb_bf16* gamma,
                                int32_t n, int32_t H, const mb_bf16* gelu_pre, mb_bf16* dx, float* dgamma,
                                float* dbeta, float* dsum, mb_stream_t s);

/* Dense GEMM on the 5th-generation tensor cores (tcgen05, TMEM accumulators, TMA-fed smem):
 *   C[M,N] = op(A) op(B)^T   with  op(A)[m,k] = a_t ? A[k*lda + m] : A[m*lda + k]
 *                                  op(B)[n,k] = b_t ? B[k*ldb + n] : B[n*ldb + k]
 * (b_t = 0 is the nn.Linear y = x W^T case; a_t = b_t = 1 is the weight-gradient dW = dY^T X.)
 * epilogue:
 *   MB_EPI_BF16      C bf16 = acc (+ bias[n]) (+ residual[m,n])
 *   MB_EPI_F32_ACC   C fp32 += acc  (atomic; enables split-K and gradient accumulation)
 *   MB_EPI_F32       C fp32 = acc (+ bias[n])
 *   MB_EPI_GELU_AUX  aux bf16 = acc + bias (pre-activation), C bf16 = GeLU(acc + bias)
 * All leading dimensions are in elements and must be multiples of 8; pointers 16-byte aligned. */
enum { MB_EPI_BF16 = 0, MB_EPI_F32_ACC = 1, MB_EPI_F32 = 2, MB_EPI_GELU_AUX = 3 };
MB_API mb_status mb_gemm(int32_t M, int32_t N, int32_t K, const mb_bf16* A, int64_t lda, int32_t a_t, const mb_bf16* B,
                  int64_t ldb, int32_t b_t, void* C, int64_t ldc, int32_t epilogue, const mb_bf16* bias,
                  const mb_bf16* residual, int64_t ldr, mb_bf16* aux, int64_t ldaux, mb_stream_t s);

/* Weight gradient with fused bias gradient (the bias of y = x W^T + b has db = sum over rows of dY):
 *   dW[M,N] += dY^T X   with dY [K, M] (lda), X [K, N] (ldb) row-major bf16, dW fp32 (ldc), and
 *   db[M] += sum_k dY[k, m]  (if db != NULL), computed on the tensor cores from the dY tiles the GEMM
 *   already stages (an extra N = 16 MMA against an all-ones tile).  Split-K partials meet in fp32
 *   atomics (+= contract). */
MB_API mb_status mb_gemm_wgrad(int32_t M, int32_t N, int32_t K, const mb_bf16* dY, int64_t lda, const mb_bf16* X,
                               int64_t ldb, float* dW, int64_t ldc, float* db, mb_stream_t s);

/* A8 — fused GLU up-projection with the GeGLU epilogue (Eq. 2; fused W1||V):
 *   U = X W_1v^T + b_1v  ([n, 2I]; first I outputs = W1 half "a", last I = V half "g", reading R8)
 *   Z = GeLU(a) * g      ([n, I], written)
 *   Gd = [g * GeLU'(a) | GeLU(a)]   ([n, 2I], written; the two factors the backward needs, so U
 *        itself never reaches memory and the backward epilogue evaluates no transcendental)
 * I must be a multiple of 128. */
MB_API mb_status mb_geglu_forward(const mb_bf16* X, int32_t n, int32_t H, int32_t I, const mb_bf16* w_1v,
                                  const mb_bf16* b_1v, mb_bf16* Gd, mb_bf16* Z, mb_stream_t s);
/* GeGLU backward fused into the dZ = dF W_2 GEMM: dZ never reaches memory;
 *   dU = dZ * Gd  i.e.  dU[:, :I] = dZ * g * GeLU'(a),  dU[:, I:] = dZ * GeLU(a)   (bf16 [n, 2I]). */
MB_API mb_status mb_geglu_backward(const mb_bf16* dF, int32_t n, int32_t H, int32_t I, const mb_bf16* w_2,
                                   const mb_bf16* Gd, mb_bf16* dU, mb_stream_t s);

/* A5 — varlen ALiBi attention forward (Eq. 1; FlashAttention P:120), on the packed
 * stream, with the bias -m_h |i-j| generated in-kernel (never materialised):
 *   s_ij = q_i . k_j / sqrt(d) - m_h |i - j|   (i, j positions inside one sequence, R2/R4)
 *   O_i = sum_j softmax_j(s)_ij v_j,  LSE_i = log sum_j exp(s_ij)
 *   qkv bf16 [nnz, 3H] with columns (3, heads, d) (R9); cu_seqlens device int32[batch+1];
 *   slopes device fp32[heads]; O bf16 [nnz, H]; lse fp32 [heads, nnz] (saved for backward).
 * max_seqlen <= 2048 (BASELINE config 4 is 512; SURVEY F4 adds 1024 and 2048). */
MB_API mb_status mb_attention_forward(const mb_bf16* qkv, const int32_t* cu_seqlens, int32_t batch, int32_t nnz,
                               int32_t max_seqlen, int32_t heads, int32_t head_dim, const float* slopes,
                               mb_bf16* O, float* lse, mb_stream_t s);
/* A10 — varlen ALiBi attention backward (recomputes P from LSE; no dropout P:152):
 *   dV = P^T dO, dP = dO V^T, dS = P (dP - D), D_i = dO_i . O_i, dQ = dS K/sqrt d, dK = dS^T Q/sqrt d
 * written into dqkv bf16 [nnz, 3H] in the qkv column layout.  If db_qkv != NULL, the column sums of
 * dqkv (the QKV-projection bias gradient) are accumulated into it (fp32 [3H], +=).
 * ws: mb_attention_workspace_bytes (non-zero for every max_seqlen: short batches with more
 * (sequence, head) units than the short kernel's per-CTA unit lists hold run on the long kernel). */
MB_API size_t mb_attention_workspace_bytes(int32_t nnz, int32_t heads, int32_t head_dim, int32_t max_seqlen);
MB_API mb_status mb_attention_backward(const mb_bf16* qkv, const mb_bf16* O, const mb_bf16* dO, const float* lse,
                                const int32_t* cu_seqlens, int32_t batch, int32_t nnz, int32_t max_seqlen,
                                int32_t heads, int32_t head_dim, const float* slopes, mb_bf16* dqkv,
                                float* db_qkv, void* ws, size_t ws_bytes, mb_stream_t s);

/* Column sums: out[c] += sum_r x[r, c] (fp32 accumulate) — bias gradients.  x bf16 [n, C]. */
MB_API mb_status mb_colsum(const mb_bf16* x, int32_t n, int32_t C, float* out, mb_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * A4-A10 — one post-LN encoder layer on the packed stream (R1):
 *   QKV = X Wqkv^T + bqkv; C = ALiBiAttn(QKV); Y1 = LN1(C Wo^T + bo + X);
 *   U = Y1 W1v^T + b1v; Z = GeLU(U_a) * U_g; Y = LN2(Z W2^T + b2 + Y1)
 * x, y: bf16 [nnz, H] packed; slopes device fp32[heads].
 * saved: device buffer of mb_layer_saved_bytes(d, nnz) bytes, written by forward and read by the
 *        matching backward (QKV, attention output, LSE, LN inputs/stats, Y1, GeGLU factors Gd, Z).
 * ws:    device workspace of mb_layer_workspace_bytes(d, nnz, max_seqlen) bytes (backward only). */
typedef struct {
  const int32_t* cu_seqlens; /* device int32[batch+1] */
  int32_t batch, nnz, max_seqlen;
} mb_packed;

typedef struct {
  const mb_bf16 *w_qkv, *b_qkv, *w_o, *b_o, *ln1_g, *ln1_b, *w_1v, *b_1v, *w_2, *b_2, *ln2_g, *ln2_b;
} mb_layer_params;
typedef struct {
  float *w_qkv, *b_qkv, *w_o, *b_o, *ln1_g, *ln1_b, *w_1v, *b_1v, *w_2, *b_2, *ln2_g, *ln2_b;
} mb_layer_grads;

/* F2 — feed-forward dropout ("we applied 0.1 dropout to the feedforward layers"; placement
 * and generator per reading R32): S1 = X + drop_0(C Wo^T + bo), S2 = Y1 + drop_1(Z W2^T + b2),
 * drop_s(v)[t, f] = v[t, f] * keep_s(t, f) / P(keep).  keep is a pure function of (seed, stream,
 * site s, packed row t, feature f): Philox-4x32-10 (Salmon et al., SC'11) with counter
 * (f >> 3, t, 2*stream + s, 0), key (seed & 0xffffffff, seed >> 32); the uniform of f is 16-bit
 * field (f & 1) of output word (f & 7) >> 1; kept iff >= thr = round(65536 p), and a kept value is
 * scaled by 1 / P(keep) = 65536 / (65536 - thr) (inverted dropout, unbiased for every p).  The
 * backward regenerates the same mask (nothing is saved).  NULL or p == 0: no dropout.  p in [0, 1). */
typedef struct {
  float p;
  uint64_t seed;   /* one per micro-step (and rank) */
  int32_t stream;  /* layer index */
} mb_dropout;

MB_API size_t mb_layer_saved_bytes(const mb_dims* d, int32_t nnz);
MB_API size_t mb_layer_workspace_bytes(const mb_dims* d, int32_t nnz, int32_t max_seqlen);

/* drop: optional F2 dropout (NULL = none).  Errors: p outside [0, 1) -> MB_ERR_INVALID_ARG. */
MB_API mb_status mb_encoder_forward(const mb_dims* d, const mb_layer_params* p, const mb_packed* pk, const float* slopes,
                             const mb_bf16* x, mb_bf16* y, void* saved, const mb_dropout* drop, mb_stream_t s);
/* dx = dL/dx; dy is consumed (used as scratch).  Gradients accumulate into g (+=).  drop must be
 * the forward's (same seed / stream / p): the masks are regenerated, not saved. */
MB_API mb_status mb_encoder_backward(const mb_dims* d, const mb_layer_params* p, const mb_packed* pk, const float* slopes,
                              const mb_bf16* x, const void* saved, mb_bf16* dy, mb_bf16* dx,
                              const mb_layer_grads* g, void* ws, size_t ws_bytes, const mb_dropout* drop,
                              mb_stream_t s);
/* The F2 keep mask of one site as bytes (1 = kept): out[t * cols + f] for t < rows, f < cols —
 * exactly what the fused epilogues apply (a test hook for bit-exact mask parity).  out: device
 * uint8 [rows, cols]; cols % 8 == 0. */
MB_API mb_status mb_dropout_mask(const mb_dropout* drop, int32_t site, int32_t rows, int32_t cols, uint8_t* out,
                                 mb_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * A3 — embedding (no position table): x0[t] = LN_e(E_tok[ids[indices[t]]] + E_type[0]).
 * ids device int32[B*L] (padded layout); x0 bf16 [nnz, H]; stats fp32 [nnz, 2] saved for backward.
 * Ids outside [0, V) (V = d->vocab) are clamped so no access leaves E_tok / d_emb; mb_unpad_index
 * reports them (MB_ERR_TOKEN_RANGE) when given the ids. */
MB_API mb_status mb_embed_forward(const mb_dims* d, const int32_t* ids, const int32_t* indices, int32_t nnz,
                           const mb_bf16* emb, const mb_bf16* type_emb, const mb_bf16* ln_g, const mb_bf16* ln_b,
                           mb_bf16* x0, float* stats, mb_stream_t s);
/* Backward: d_emb[id] += dv, d_type_emb[0] += sum dv, d_ln_g/d_ln_b += (fp32).  dx0 is consumed.
 * ws: device workspace of mb_embed_workspace_bytes(d, nnz) bytes (0 unless d->flags has
 * MB_FLAG_DETERMINISTIC: then the dv rows, the (id, token) sort keys and the LN column partials). */
MB_API size_t mb_embed_workspace_bytes(const mb_dims* d, int32_t nnz);
MB_API mb_status mb_embed_backward(const mb_dims* d, const int32_t* ids, const int32_t* indices, int32_t nnz,
                            const mb_bf16* emb, const mb_bf16* type_emb, const mb_bf16* ln_g, const float* stats,
                            mb_bf16* dx0, float* d_emb, float* d_type_emb, float* d_ln_g, float* d_ln_b, void* ws,
                            size_t ws_bytes, mb_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * A11 — sparse MLM head + softmax cross-entropy on the masked tokens only (P:150 30% MLM; vocab
 * 30528 P:174; tied decoder R15; mean over labelled positions S:534, normalised by inv_norm = 1/N
 * with N the GLOBAL masked count of the optimizer step, R18):
 *   h_k = Y[masked_rows[k]]; t_k = GeLU(h_k W_t^T + b_t); u_k = LN_h(t_k); z_k = u_k E^T + b_dec
 *   loss_sum += inv_norm * sum_k (logsumexp(z_k) - z_k[label_k])
 * Forward and backward in one call: dy_top (bf16 [nnz, H]) is fully written (zero on unmasked rows);
 * grads accumulate (+=).  loss_sum: device fp32 scalar (+=).  lse: device fp32[n_masked] out.
 * ws: mb_mlm_workspace_bytes(d, n_masked).  dy_top == NULL and g == NULL: forward only (evaluation,
 * e.g. SURVEY F4's "train short, test long" at l up to 2048): loss_sum and lse, no gradients; only
 * one of the two NULL -> MB_ERR_INVALID_ARG. */
typedef struct {
  const mb_bf16 *w_t, *b_t, *ln_g, *ln_b, *emb /*[V,H], tied*/, *b_dec;
} mb_head_params;
typedef struct {
  float *w_t, *b_t, *ln_g, *ln_b, *emb /*[V,H], shared with the embedding*/, *b_dec;
} mb_head_grads;
MB_API size_t mb_mlm_workspace_bytes(const mb_dims* d, int32_t n_masked);
MB_API mb_status mb_mlm_loss(const mb_dims* d, const mb_head_params* p, const mb_bf16* y, int32_t nnz,
                      const int32_t* masked_rows, const int32_t* labels, int32_t n_masked, float inv_norm,
                      float* loss_sum, float* lse, mb_bf16* dy_top, const mb_head_grads* g, void* ws,
                      size_t ws_bytes, mb_stream_t s);

/* R18 loss normaliser ("mean over labelled positions"; the mean is over the GLOBAL masked count
 * N of the optimizer step): inv_out = 1 / max(N, 1), loss_out = loss_sum * inv_out, with N read from
 * the device scalar `count` (mb_mlm_select's count_accum, allreduced over ranks) or, if count is
 * NULL, the host value count_host.  Device fp32 scalars; either output may be NULL (not both). */
MB_API mb_status mb_loss_normalize(const float* loss_sum, const float* count, float count_host, float* inv_out,
                                   float* loss_out, mb_stream_t s);

/* Zero-fill of an fp32 device buffer (n elements; caller-owned): the gradient buckets and scalars
 * reset at the start of each optimizer step (the += contract of the backward calls, R18's count).
 * p may have any 4-byte alignment; n == 0 is a no-op. */
MB_API mb_status mb_zero_f32(float* p, int64_t n, mb_stream_t s);

/* F1 learning-rate schedule (Table A1; reading R34), host function: lr at
 * optimizer step `step` of `total_steps`: linear warmup 0 -> lr_peak over the first 6 % of the
 * steps, then linear decay to 0.02 lr_peak at total_steps (step clamped to [0, total_steps]);
 * lr_peak itself if total_steps <= 0.  The AdamW decay factor for that step is
 * (lr / lr_peak) * weight_decay (mb_adamw_step's weight_decay argument). */
MB_API double mb_lr_schedule(int64_t step, int64_t total_steps, double lr_peak);

/* ---------------------------------------------------------------------------------------------
 * F1 — fused decoupled AdamW update (Table A1: beta=(0.9,0.98), eps=1e-6, wd 1e-5):
 *   g' = grad_scale g; m = b1 m + (1-b1) g'; v = b2 v + (1-b2) g'^2;
 *   m_hat = m / (1 - b1^step); v_hat = v / (1 - b2^step);
 *   p = p - lr m_hat / (sqrt(v_hat) + eps) - weight_decay p
 * "Decoupled" (reading R34, Loshchilov & Hutter): the decay never enters the gradient and is NOT
 * multiplied by lr; weight_decay is the per-step factor (lr_t / lr_peak) * wd that the caller
 * derives from the schedule (warmup 6 %, linear decay to 0.02 lr).
 * master fp32 [n] in/out, m, v fp32 [n] in/out, g fp32 [n], w_bf16 [n] out (RNE of the new master:
 * the bf16 weight copy the kernels read).  step >= 1.  Stream-ordered, allocates nothing.
 * Errors: NULL pointer, n < 0 or step < 1 -> MB_ERR_INVALID_ARG; launch failure -> MB_ERR_CUDA. */
MB_API mb_status mb_adamw_step(float* master, float* m, float* v, const float* g, mb_bf16* w_bf16, int64_t n, float lr,
                        float beta1, float beta2, float eps, float weight_decay, float grad_scale, int32_t step,
                        mb_stream_t s);
/* The same update with the gradient scale read from DEVICE memory: g' = grad_scale * (*grad_scale_dev) g.
 * Lets a data-parallel step normalise by the global masked-token count (R18) that an in-stream
 * allreduce produced, without reading it back to the host.  grad_scale_dev: device fp32 scalar. */
MB_API mb_status mb_adamw_step_dev(float* master, float* m, float* v, const float* g, mb_bf16* w_bf16, int64_t n,
                            float lr, float beta1, float beta2, float eps, float weight_decay, float grad_scale,
                            const float* grad_scale_dev, int32_t step, mb_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * F3 — baselines for the paper's throughput ablations; not on the training path.
 *
 * fp32 LayerNorm (the alternative to P:145's bf16 LN, "only 2-bytes are required per-element"):
 * the same forward / backward as mb_layernorm_forward / _backward with fp32 x, y, dy, dx
 * [n, H] (gamma, beta bf16 as in the model).  Backward requires H % 256 == 0.  dsum may be NULL.
 * Errors: NULL pointer / negative size -> MB_ERR_INVALID_ARG; H % 8 (fwd), H % 256 (bwd) or
 * H > 1024 -> MB_ERR_CONFIG. */
MB_API mb_status mb_layernorm_forward_f32(const float* x, const mb_bf16* gamma, const mb_bf16* beta, int32_t n,
                                          int32_t H, float eps, float* y, float* stats, mb_stream_t s);
MB_API mb_status mb_layernorm_backward_f32(const float* dy, const float* x, const float* stats,
                                           const mb_bf16* gamma, int32_t n, int32_t H, float* dx, float* dgamma,
                                           float* dbeta, float* dsum, mb_stream_t s);
/* Naive (unfused) GLU, elementwise halves (Eq. 2): with U_a = x W1^T + b1 and
 * U_g = x V^T + b_v computed by two separate mb_gemm calls,
 *   forward:  Z = GeLU(U_a) * U_g                                  (exact-erf GeLU, R7)
 *   backward: dU_a = dZ * U_g * GeLU'(U_a),  dU_g = dZ * GeLU(U_a)
 * All bf16, `count` elements each (count % 8 == 0, contiguous). */
MB_API mb_status mb_geglu_naive_forward(const mb_bf16* ua, const mb_bf16* ug, int64_t count, mb_bf16* z,
                                        mb_stream_t s);
MB_API mb_status mb_geglu_naive_backward(const mb_bf16* dz, const mb_bf16* ua, const mb_bf16* ug, int64_t count,
                                         mb_bf16* dua, mb_bf16* dug, mb_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* MOSAICBERT_H_ */
