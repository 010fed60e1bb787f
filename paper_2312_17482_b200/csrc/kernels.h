// Internal launcher interface shared by the C-ABI composites (api.cu) and the kernel files.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace mb {

constexpr int kMaxSeqlen = 2048;  // longest sequence the attention kernels accept (F4)


enum EpiMode { E_BF16 = 0, E_F32_ACC = 1, E_F32 = 2, E_GELU_AUX = 3, E_GEGLU_FWD = 4, E_GEGLU_BWD = 5, E_LSE = 6, E_DZ = 7 };

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
};

mb_status gemm(const GemmArgs& g, cudaStream_t s);

mb_status layernorm_fwd(const bf16* x, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                        float* stats, cudaStream_t s);
// drop.thr > 0 (F2 backward): dx = dL/d(LN input) (the residual path) and dxd = dx * keep * scale
// (the gradient of the dropped projection output); dsum then sums dxd
mb_status layernorm_bwd(const bf16* dy, const bf16* x, const float* stats, const bf16* gamma, int n, int H,
                        const bf16* gelu_pre, bf16* dx, float* dgamma, float* dbeta, float* dsum, cudaStream_t s,
                        const DropArgs* drop = nullptr, bf16* dxd = nullptr);
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
};
mb_status embed_ln_fwd(const EmbedSrc& e, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                       float* stats, cudaStream_t s);
mb_status embed_ln_bwd(const EmbedSrc& e, const bf16* dy, const float* stats, const bf16* gamma, int n, int H,
                       float* dgamma, float* dbeta, float* dsum, cudaStream_t s);
mb_status colsum(const bf16* x, int n, int C, float* out, cudaStream_t s);

mb_status attention_fwd(const bf16* qkv, const int* cu, int batch, int nnz, int max_seqlen, int heads, int d,
                        const float* slopes, bf16* O, float* lse, cudaStream_t s);
size_t attention_ws_bytes(int nnz, int heads, int d, int max_seqlen);
mb_status attention_bwd(const bf16* qkv, const bf16* O, const bf16* dO, const float* lse, const int* cu, int batch,
                        int nnz, int max_seqlen, int heads, int d, const float* slopes, bf16* dqkv, float* dbias,
                        void* ws, size_t ws_bytes, cudaStream_t s);

}  // namespace mb
