// A4-A10 — one post-LN MosaicBERT encoder layer on the unpadded stream,
// forward and backward, composed from the tcgen05 GEMMs (fused epilogues), the varlen ALiBi
// attention kernels and the bf16 LayerNorm kernels.  Host code only: it validates arguments, carves
// the caller's `saved` / workspace buffers and enqueues kernels on the caller's stream.
#include <algorithm>
#include "common.cuh"
#include "kernels.h"

namespace mb {
namespace {

inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct Saved {  // written by forward, read by backward
  bf16 *qkv, *o, *s1, *y1, *u, *z, *s2;
  float *lse, *st1, *st2;
  size_t bytes;
  Saved(char* base, int T, int H, int I, int heads) {
    size_t off = 0;
    auto take = [&](size_t b) {
      char* p = base ? base + off : nullptr;
      off += al(b);
      return p;
    };
    qkv = (bf16*)take((size_t)T * 3 * H * 2);
    o = (bf16*)take((size_t)T * H * 2);
    lse = (float*)take((size_t)heads * T * 4);
    s1 = (bf16*)take((size_t)T * H * 2);
    st1 = (float*)take((size_t)T * 8);
    y1 = (bf16*)take((size_t)T * H * 2);
    u = (bf16*)take((size_t)T * 2 * I * 2);
    z = (bf16*)take((size_t)T * I * 2);
    s2 = (bf16*)take((size_t)T * H * 2);
    st2 = (float*)take((size_t)T * 8);
    bytes = off;
  }
};

struct Ws {  // backward scratch
  bf16 *ds2, *du, *dy1, *ds1, *dO, *dqkv;
  void* attn;
  size_t attn_bytes, bytes;
  Det det;  // deterministic mode (MB_FLAG_DETERMINISTIC): partial slab + split-K turnstiles
  Ws(char* base, int T, int H, int I, int heads, int max_seqlen, bool deterministic) {
    size_t off = 0;
    auto take = [&](size_t b) {
      char* p = base ? base + off : nullptr;
      off += al(b);
      return p;
    };
    ds2 = (bf16*)take((size_t)T * H * 2);
    du = (bf16*)take((size_t)T * 2 * I * 2);
    dy1 = (bf16*)take((size_t)T * H * 2);
    ds1 = (bf16*)take((size_t)T * H * 2);
    dO = (bf16*)take((size_t)T * H * 2);
    dqkv = (bf16*)take((size_t)T * 3 * H * 2);
    attn_bytes = attention_ws_bytes(T, heads, H / heads, max_seqlen, deterministic);
    attn = take(attn_bytes);
    if (deterministic) {
      det.part_floats = std::max({layernorm_bwd_det_floats(T, H), gemm_det_floats(2 * I, H, T), colsum_det_floats(T, H)});
      det.part = (float*)take(det.part_floats * 4);
      det.sem_count = std::max({gemm_det_sems(H, I), gemm_det_sems(2 * I, H), gemm_det_sems(H, H), gemm_det_sems(3 * H, H)});
      det.sem = (int*)take((size_t)det.sem_count * 4);
      if (!base) det.part = nullptr;
    }
    bytes = off;
  }
};

inline bool det_of(const mb_dims* d) { return d && (d->flags & MB_FLAG_DETERMINISTIC); }

mb_status check_dims(const mb_dims* d) {
  if (!d) return MB_ERR_INVALID_ARG;
  if (d->heads <= 0 || d->hidden <= 0 || d->hidden % d->heads) return MB_ERR_CONFIG;
  const int hd = d->hidden / d->heads;
  if (hd != 32 && hd != 64) return MB_ERR_CONFIG;
  if (d->hidden % 8 || d->hidden > 1024 || d->intermediate % 128 || d->intermediate <= 0) return MB_ERR_CONFIG;
  return MB_OK;
}

inline const bf16* B(const mb_bf16* p) { return reinterpret_cast<const bf16*>(p); }

bool drop_ok(const mb_dropout* dr) { return !dr || (dr->p >= 0.f && dr->p < 1.f && dr->stream >= 0); }

__global__ void dropout_mask_kernel(DropArgs d, int rows, int cols, uint8_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 8-feature group
  const int gpr = cols / 8;
  if (i >= (int64_t)rows * gpr) return;
  const int t = (int)(i / gpr), f0 = (int)(i - (int64_t)t * gpr) * 8;
  const uint32_t bits = dropout_keep8(d, (uint32_t)t, (uint32_t)f0);
  uint2 v;
  v.x = (bits & 1u) | ((bits >> 1) & 1u) << 8 | ((bits >> 2) & 1u) << 16 | ((bits >> 3) & 1u) << 24;
  v.y = ((bits >> 4) & 1u) | ((bits >> 5) & 1u) << 8 | ((bits >> 6) & 1u) << 16 | ((bits >> 7) & 1u) << 24;
  *reinterpret_cast<uint2*>(out + (int64_t)t * cols + f0) = v;
}

}  // namespace

// F2 (R32): host-side dropout parameters of one site; thr = 0 (off) for NULL / p == 0
DropArgs make_drop_args(const mb_dropout* dr, int site) {
  DropArgs a;
  if (!dr || dr->p <= 0.f) return a;
  a.key0 = (uint32_t)(dr->seed & 0xFFFFFFFFull);
  a.key1 = (uint32_t)(dr->seed >> 32);
  a.site = 2u * (uint32_t)dr->stream + (uint32_t)site;
  a.thr = (uint32_t)std::lround((double)dr->p * 65536.0);
  // inverted dropout: the scale is 1 / P(keep) with P(keep) = (65536 - thr) / 65536 exactly, so
  // E[drop(v)] = v for every p (not only those with 65536 p integral)
  a.scale = (float)(65536.0 / (65536.0 - (double)a.thr));
  return a;
}

}  // namespace mb

extern "C" {

size_t mb_layer_saved_bytes(const mb_dims* d, int32_t nnz) {
  if (!d || d->heads <= 0) return 0;
  return mb::Saved(nullptr, std::max(nnz, 1), d->hidden, d->intermediate, d->heads).bytes;
}

size_t mb_layer_workspace_bytes(const mb_dims* d, int32_t nnz, int32_t max_seqlen) {
  if (!d || d->heads <= 0) return 0;
  return mb::Ws(nullptr, std::max(nnz, 1), d->hidden, d->intermediate, d->heads, max_seqlen, mb::det_of(d)).bytes;
}

mb_status mb_dropout_mask(const mb_dropout* drop, int32_t site, int32_t rows, int32_t cols, uint8_t* out,
                          mb_stream_t s_) {
  using namespace mb;
  if (!drop || !out || rows < 0 || cols < 0 || site < 0 || site > 1 || !drop_ok(drop)) return MB_ERR_INVALID_ARG;
  if (cols % 8) return MB_ERR_CONFIG;
  if (rows == 0 || cols == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  const int64_t groups = (int64_t)rows * (cols / 8);
  dropout_mask_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(s_)>>>(
      make_drop_args(drop, site), rows, cols, out);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_encoder_forward(const mb_dims* d, const mb_layer_params* p, const mb_packed* pk, const float* slopes,
                             const mb_bf16* x, mb_bf16* y, void* saved, const mb_dropout* drop, mb_stream_t s_) {
  using namespace mb;
  mb_status st = check_dims(d);
  if (st != MB_OK) return st;
  if (!p || !pk || !slopes || !x || !y || !saved || !pk->cu_seqlens || !drop_ok(drop)) return MB_ERR_INVALID_ARG;
  if (pk->nnz < 0 || pk->batch < 0) return MB_ERR_INVALID_ARG;
  if (pk->max_seqlen > kMaxSeqlen) return MB_ERR_SHAPE;
  if (pk->nnz == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(s_);
  const int T = pk->nnz, H = d->hidden, I = d->intermediate, nh = d->heads;
  Saved sv(reinterpret_cast<char*>(saved), T, H, I, nh);
#define TRY(e)                          \
  do {                                  \
    if ((st = (e)) != MB_OK) return st; \
  } while (0)
  {  // A4: QKV = X Wqkv^T + bqkv
    GemmArgs a;
    a.M = T, a.N = 3 * H, a.K = H, a.A = B(x), a.lda = H, a.B = B(p->w_qkv), a.ldb = H;
    a.ep.mode = E_BF16, a.ep.C = sv.qkv, a.ep.ldc = 3 * H, a.ep.bias = B(p->b_qkv);
    TRY(gemm(a, s));
  }
  // A5: varlen ALiBi attention
  probe_begin(PROBE_ATTN_FWD, s);
  TRY(attention_fwd(sv.qkv, pk->cu_seqlens, pk->batch, T, pk->max_seqlen, nh, H / nh, slopes, sv.o, sv.lse, s));
  probe_end(PROBE_ATTN_FWD, s);
  {  // A6: S1 = O Wo^T + bo + X
    GemmArgs a;
    a.M = T, a.N = H, a.K = H, a.A = sv.o, a.lda = H, a.B = B(p->w_o), a.ldb = H;
    a.ep.mode = E_BF16, a.ep.C = sv.s1, a.ep.ldc = H, a.ep.bias = B(p->b_o), a.ep.res = B(x), a.ep.ldr = H;
    a.ep.drop = make_drop_args(drop, 0);  // F2 site 0: S1 = X + drop(O Wo^T + bo)
    TRY(gemm(a, s));
  }
  // A7: Y1 = LN1(S1)
  probe_begin(PROBE_LN_FWD, s);
  TRY(layernorm_fwd(sv.s1, B(p->ln1_g), B(p->ln1_b), T, H, d->ln_eps, sv.y1, sv.st1, s));
  probe_end(PROBE_LN_FWD, s);
  {  // A8: U = Y1 W1v^T + b1v, Z = GeLU(U_a) * U_g; saves Gd = [U_g GeLU'(U_a) | GeLU(U_a)] in sv.u
    GemmArgs a;
    a.M = T, a.N = 2 * I, a.K = H, a.A = sv.y1, a.lda = H, a.B = B(p->w_1v), a.ldb = H;
    a.ep.mode = E_GEGLU_FWD, a.ep.C = sv.z, a.ep.ldc = I, a.ep.bias = B(p->b_1v), a.ep.aux = sv.u,
    a.ep.ldaux = 2 * I, a.ep.I = I;
    probe_begin(PROBE_GEGLU_FWD, s);
    TRY(gemm(a, s));
    probe_end(PROBE_GEGLU_FWD, s);
  }
  {  // A9: S2 = Z W2^T + b2 + Y1
    GemmArgs a;
    a.M = T, a.N = H, a.K = I, a.A = sv.z, a.lda = I, a.B = B(p->w_2), a.ldb = I;
    a.ep.mode = E_BF16, a.ep.C = sv.s2, a.ep.ldc = H, a.ep.bias = B(p->b_2), a.ep.res = sv.y1, a.ep.ldr = H;
    a.ep.drop = make_drop_args(drop, 1);  // F2 site 1: S2 = Y1 + drop(Z W2^T + b2)
    TRY(gemm(a, s));
  }
  // A7: Y = LN2(S2)
  TRY(layernorm_fwd(sv.s2, B(p->ln2_g), B(p->ln2_b), T, H, d->ln_eps, reinterpret_cast<bf16*>(y), sv.st2, s));
  return MB_OK;
}

mb_status mb_encoder_backward(const mb_dims* d, const mb_layer_params* p, const mb_packed* pk, const float* slopes,
                              const mb_bf16* x, const void* saved, mb_bf16* dy, mb_bf16* dx, const mb_layer_grads* g,
                              void* ws, size_t ws_bytes, const mb_dropout* drop, mb_stream_t s_) {
  using namespace mb;
  mb_status st = check_dims(d);
  if (st != MB_OK) return st;
  if (!p || !pk || !slopes || !x || !saved || !dy || !dx || !g || !ws || !pk->cu_seqlens || !drop_ok(drop))
    return MB_ERR_INVALID_ARG;
  if (pk->nnz < 0 || pk->batch < 0) return MB_ERR_INVALID_ARG;
  if (pk->max_seqlen > kMaxSeqlen) return MB_ERR_SHAPE;
  if (pk->nnz == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(s_);
  const int T = pk->nnz, H = d->hidden, I = d->intermediate, nh = d->heads;
  Saved sv(reinterpret_cast<char*>(const_cast<void*>(saved)), T, H, I, nh);
  Ws w(reinterpret_cast<char*>(ws), T, H, I, nh, pk->max_seqlen, det_of(d));
  if (ws_bytes < w.bytes) return MB_ERR_WORKSPACE;
  const Det* det = w.det ? &w.det : nullptr;
  // the turnstiles start at zero (each GEMM's last split resets its own counters)
  if (det && cudaMemsetAsync(w.det.sem, 0, (size_t)w.det.sem_count * 4, s) != cudaSuccess) return MB_ERR_CUDA;
  // F2: with dropout the projection branches see dF = dS2 * keep / (1 - p) (dp2) and dA = dS1 * keep
  // / (1 - p) (dp1), while the residual branches keep dS2 / dS1.  dp2 lives in w.dy1 (written only
  // after its last reader, dW2) and dp1 in the front of w.dqkv (written only by the attention
  // backward, after dWo).  Without dropout dp = dS.
  const DropArgs dr2 = make_drop_args(drop, 1), dr1 = make_drop_args(drop, 0);
  bf16* dp2 = dr2.thr ? w.dy1 : w.ds2;
  bf16* dp1 = dr1.thr ? w.dqkv : w.ds1;
  // LN2 backward: dS2 (and dp2); dgamma2, dbeta2; db2 = column sums of dp2 (same pass)
  TRY(layernorm_bwd(reinterpret_cast<bf16*>(dy), sv.s2, sv.st2, B(p->ln2_g), T, H, nullptr, w.ds2, g->ln2_g,
                    g->ln2_b, g->b_2, s, &dr2, dr2.thr ? dp2 : nullptr, det));
  {  // dZ = dF W2 fused with the GeGLU backward -> dU = dZ * Gd = [dZ g GeLU'(a) | dZ GeLU(a)]
    GemmArgs a;
    a.M = T, a.N = I, a.K = H, a.A = dp2, a.lda = H, a.B = B(p->w_2), a.ldb = I, a.b_t = true;
    a.ep.mode = E_GEGLU_BWD, a.ep.C = w.du, a.ep.ldc = 2 * I, a.ep.U = sv.u, a.ep.ldu = 2 * I, a.ep.I = I;
    TRY(gemm(a, s));
  }
  {  // dW2 += dF^T Z
    GemmArgs a;
    a.M = H, a.N = I, a.K = T, a.A = dp2, a.lda = H, a.a_t = true, a.B = sv.z, a.ldb = I, a.b_t = true;
    a.ep.mode = E_F32_ACC, a.ep.C = g->w_2, a.ep.ldc = I;
    a.det = det;
    TRY(gemm(a, s));
  }
  {  // dY1 = dU W1v + dS2
    GemmArgs a;
    a.M = T, a.N = H, a.K = 2 * I, a.A = w.du, a.lda = 2 * I, a.B = B(p->w_1v), a.ldb = H, a.b_t = true;
    a.ep.mode = E_BF16, a.ep.C = w.dy1, a.ep.ldc = H, a.ep.res = w.ds2, a.ep.ldr = H;
    TRY(gemm(a, s));
  }
  {  // dW1v += dU^T Y1; db1v += dU^T 1 (column sums of dU) by an extra N=16 MMA in the same k-loop
    GemmArgs a;
    a.M = 2 * I, a.N = H, a.K = T, a.A = w.du, a.lda = 2 * I, a.a_t = true, a.B = sv.y1, a.ldb = H, a.b_t = true;
    a.ep.mode = E_F32_ACC, a.ep.C = g->w_1v, a.ep.ldc = H, a.ep.dbias = g->b_1v;
    a.det = det;
    TRY(gemm(a, s));
  }
  // LN1 backward: dS1 (and dp1); dgamma1, dbeta1; dbo = column sums of dp1 (same pass)
  TRY(layernorm_bwd(w.dy1, sv.s1, sv.st1, B(p->ln1_g), T, H, nullptr, w.ds1, g->ln1_g, g->ln1_b, g->b_o, s, &dr1,
                    dr1.thr ? dp1 : nullptr, det));
  {  // dO = dA Wo
    GemmArgs a;
    a.M = T, a.N = H, a.K = H, a.A = dp1, a.lda = H, a.B = B(p->w_o), a.ldb = H, a.b_t = true;
    a.ep.mode = E_BF16, a.ep.C = w.dO, a.ep.ldc = H;
    TRY(gemm(a, s));
  }
  {  // dWo += dA^T O
    GemmArgs a;
    a.M = H, a.N = H, a.K = T, a.A = dp1, a.lda = H, a.a_t = true, a.B = sv.o, a.ldb = H, a.b_t = true;
    a.ep.mode = E_F32_ACC, a.ep.C = g->w_o, a.ep.ldc = H;
    a.det = det;
    TRY(gemm(a, s));
  }
  // A10: attention backward -> dQKV
  probe_begin(PROBE_ATTN_BWD, s);
  TRY(attention_bwd(sv.qkv, sv.o, w.dO, sv.lse, pk->cu_seqlens, pk->batch, T, pk->max_seqlen, nh, H / nh, slopes,
                    w.dqkv, g->b_qkv, w.attn, w.attn_bytes, s, det));  // also dbqkv = column sums of dQKV
  probe_end(PROBE_ATTN_BWD, s);
  {  // dX = dQKV Wqkv + dS1
    GemmArgs a;
    a.M = T, a.N = H, a.K = 3 * H, a.A = w.dqkv, a.lda = 3 * H, a.B = B(p->w_qkv), a.ldb = H, a.b_t = true;
    a.ep.mode = E_BF16, a.ep.C = dx, a.ep.ldc = H, a.ep.res = w.ds1, a.ep.ldr = H;
    TRY(gemm(a, s));
  }
  {  // dWqkv += dQKV^T X
    GemmArgs a;
    a.M = 3 * H, a.N = H, a.K = T, a.A = w.dqkv, a.lda = 3 * H, a.a_t = true, a.B = B(x), a.ldb = H, a.b_t = true;
    a.ep.mode = E_F32_ACC, a.ep.C = g->w_qkv, a.ep.ldc = H;
    a.det = det;
    TRY(gemm(a, s));
  }
#undef TRY
  return MB_OK;
}

}  // extern "C"
