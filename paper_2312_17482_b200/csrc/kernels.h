// Internal launcher interface shared by the C-ABI composites (api.cu) and the kernel files.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace mb {

constexpr int kMaxSeqlen = 2048;  // longest sequence the attention kernels accept (F4)


enum EpiMode { E_BF16 = 0, E_F32_ACC = 1, E_F32 = 2, E_GELU_AUX = 3, E_GEGLU_FWD = 4, E_GEGLU_BWD = 5, E_LSE = 6, E_DZ = 7 };

// Deterministic reductions (mb_dims.flags & MB_FLAG_DETERMINISTIC): fp32 sums that
// several CTAs contribute to are written as per-CTA / per-split partials into `part` and summed in a
// fixed order by ordered_sum(); split-K weight-gradient tiles are accumulated split by split in
// split order, serialised by per-tile turnstile counters `sem` (zero between uses; the last split
// resets them).  nullptr everywhere = fp32 atomics (the fast default).
struct Det {
  float* part = nullptr;
  size_t part_floats = 0;
  int* sem = nullptr;
  int sem_count = 0;
  explicit operator bool() const { return part != nullptr; }
};

struct Epi {
  int mode = E_BF16;
  void* C = nullptr;            // output (bf16 or fp32, per mode)
  int64_t ldc = 0;
  const bf16* bias = nullptr;   // [N] (GEGLU_FWD: [2I])
  const bf16* res = nullptr;    // residual [M, N] (E_BF16)
  int64_t ldr = 0;
  bf16* aux = nullptr;          // GELU_AUX: pre-activation out; GEGLU_FWD: Gd out [M, 2I]
  int64_t ldaux = 0;
  const bf16* U = nullptr;      // GEGLU_BWD: saved Gd = [g GeLU'(a) | GeLU(a)] [M, 2I]
  int64_t ldu = 0;
  int I = 0;                    // GeGLU half width
  float* dbias = nullptr;       // GEGLU_BWD: column sums of dU accumulated here (fp32 [2I], +=)
  // fused softmax-cross-entropy over the columns (decoder GEMM, A11):
  //   E_LSE: per row and (tile, column half) the online (max, sum exp) of z = acc + bias -> part,
  //          and the label logit -> zlab;   E_DZ: C = bf16((exp(z - lse[row]) - [col == label]) * inv_norm)
  const int* labels = nullptr;
  const float* lse = nullptr;
  float2* part = nullptr;
  float* zlab = nullptr;
  int npart = 0;
  float inv_norm = 1.f;
  // F2 dropout between bias and residual (E_BF16 with drop.thr > 0; compiled into one variant)
  DropArgs drop;
  // deterministic mode: E_F32_ACC split-K turnstile counters (one per tile and CTA of the pair) and
  // the bias-gradient partial slab [splits * num_n, M] (ACC == 1 kernels)
  int* sem = nullptr;
  float* dpart = nullptr;
  // E_BF16: the output leaves by TMA stores through tmC (host-checked: 16-byte aligned C, ldc % 8 == 0,
  // and with NSCR == 1 no residual, whose staging would share the single scratch block)
  int tma_store = 0;
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const bf16* A = nullptr;
  int64_t lda = 0;
  bool a_t = false;  // false: A[m*lda + k]; true: A[k*lda + m]
  const bf16* B = nullptr;
  int64_t ldb = 0;
  bool b_t = false;  // false: B[n*ldb + k]; true: B[k*ldb + n]
  Epi ep;
  const Det* det = nullptr;  // deterministic mode (E_F32_ACC split-K order, fused bias-gradient partials)
};

mb_status gemm(const GemmArgs& g, cudaStream_t s);
// deterministic-mode workspace of one E_F32_ACC GEMM: db partial floats and turnstile counters
size_t gemm_det_floats(int M, int N, int K);
int gemm_det_sems(int M, int N);

mb_status layernorm_fwd(const bf16* x, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                        float* stats, cudaStream_t s);
// drop.thr > 0 (F2 backward): dx = dL/d(LN input) (the residual path) and dxd = dx * keep * scale
// (the gradient of the dropped projection output); dsum then sums dxd
mb_status layernorm_bwd(const bf16* dy, const bf16* x, const float* stats, const bf16* gamma, int n, int H,
                        const bf16* gelu_pre, bf16* dx, float* dgamma, float* dbeta, float* dsum, cudaStream_t s,
                        const DropArgs* drop = nullptr, bf16* dxd = nullptr, const Det* det = nullptr);
// floats of `part` the LN backward needs in deterministic mode (per-CTA partials of dgamma, dbeta, dsum)
size_t layernorm_bwd_det_floats(int n, int H);
DropArgs make_drop_args(const mb_dropout* d, int site);
mb_status gather_rows(const bf16* src, const int* idx, int n, int H, bf16* dst, cudaStream_t s);
mb_status scatter_rows(const bf16* src, const int* idx, int n, int H, int rows, bf16* dst, cudaStream_t s);

// embedding LN: x = emb[ids[indices[t]]] + type_emb[0] is recomputed inside the LN kernels
struct EmbedSrc {
  const int* ids = nullptr;
  const int* indices = nullptr;
  const bf16* emb = nullptr;
  const bf16* type_emb = nullptr;
  float* d_emb = nullptr;  // backward: dv is red-added into d_emb[id]
  int vocab = 1;           // ids are clamped to [0, vocab)
  float* dv_out = nullptr;      // deterministic mode: dv rows fp32 [n, H] (embed_det_bytes)
  unsigned long long* keys = nullptr;  // deterministic mode: sort keys [pow2 >= n]
};
// deterministic embedding scatter: d_emb[id] += sum over the tokens t with ids[indices[t]] == id of
// dv[t], in ascending t (bitonic sort of (id, t) keys, then one CTA per id)
mb_status embed_scatter_det(const float* dv, const int* ids, const int* indices, int n, int H, int vocab,
                            unsigned long long* keys, float* d_emb, cudaStream_t s);
size_t embed_det_bytes(int n, int H);
mb_status embed_ln_fwd(const EmbedSrc& e, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                       float* stats, cudaStream_t s);
mb_status embed_ln_bwd(const EmbedSrc& e, const bf16* dy, const float* stats, const bf16* gamma, int n, int H,
                       float* dgamma, float* dbeta, float* dsum, cudaStream_t s, const Det* det = nullptr);
mb_status colsum(const bf16* x, int n, int C, float* out, cudaStream_t s);
// deterministic column sums out[c] += sum_r x[r * ldx + c0 + c], c < C (fixed row chunks, ordered
// second pass); part needs colsum_det_floats(n, C) floats
size_t colsum_det_floats(int n, int C);
mb_status colsum_det(const bf16* x, int64_t ldx, int n, int C, float* out, float* part, cudaStream_t s);
// out[c] += sum_{p < nparts} part[p * stride + c] in order p = 0, 1, ... (c < count)
mb_status ordered_sum(const float* part, int nparts, int64_t stride, int count, float* out, cudaStream_t s);

mb_status attention_fwd(const bf16* qkv, const int* cu, int batch, int nnz, int max_seqlen, int heads, int d,
                        const float* slopes, bf16* O, float* lse, cudaStream_t s);
size_t attention_ws_bytes(int nnz, int heads, int d, int max_seqlen, bool det = false);
mb_status attention_bwd(const bf16* qkv, const bf16* O, const bf16* dO, const float* lse, const int* cu, int batch,
                        int nnz, int max_seqlen, int heads, int d, const float* slopes, bf16* dqkv, float* dbias,
                        void* ws, size_t ws_bytes, cudaStream_t s, const Det* det = nullptr);

}  // namespace mb
