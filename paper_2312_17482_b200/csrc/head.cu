// A11 — sparse MLM head on the masked tokens only + softmax cross-entropy ("30% masking
// ratio"; vocab 30528 P:174; tied decoder R15; loss = mean over labelled positions S:534 with the
// global count R18), A3 embedding composites, and the F1 fused AdamW step.
#include <algorithm>
#include "common.cuh"
#include "kernels.h"

namespace mb {
namespace {

// combine the per-(tile, half) online softmax partials of a row: LSE and the row loss
__global__ void ce_combine_kernel(const float2* __restrict__ part, int npart, const float* __restrict__ zlab, int n,
                                  float* __restrict__ lse_out, float* __restrict__ row_loss) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  constexpr float L2E = 1.4426950408889634f;
  float m = -INFINITY, s = 0.f;
  for (int i = lane; i < npart; i += 32) {
    const float2 p = part[(int64_t)row * npart + i];
    if (p.y > 0.f) {
      const float nm = fmaxf(m, p.x);
      s = s * exp2f((m - nm) * L2E) + p.y * exp2f((p.x - nm) * L2E);
      m = nm;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const float os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, om);
    s = (s > 0.f ? s * exp2f((m - nm) * L2E) : 0.f) + (os > 0.f ? os * exp2f((om - nm) * L2E) : 0.f);
    m = nm;
  }
  if (lane == 0) {
    const float l = m + logf(s);
    lse_out[row] = l;
    row_loss[row] = l - zlab[row];
  }
}

__global__ void sum_kernel(const float* __restrict__ x, int n, float scale, float* __restrict__ out) {
  __shared__ float sw[32];
  float t = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += x[i];
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    float u = threadIdx.x < (blockDim.x >> 5) ? sw[threadIdx.x] : 0.f;
    u = warp_sum(u);
    if (threadIdx.x == 0) *out += u * scale;
  }
}

// R18: the step's loss and gradient scale from the device-resident global masked count
// fp32 zero fill: the unaligned head element-wise, the aligned body in 16-byte stores, the tail
__global__ void zero_f32_kernel(float* __restrict__ p, int64_t n, int64_t head, int64_t n4) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
  if (tid < head) p[tid] = 0.f;
  float4* q = reinterpret_cast<float4*>(p + head);
  for (int64_t i = tid; i < n4; i += step) q[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t t0 = head + 4 * n4;
  if (tid < n - t0) p[t0 + tid] = 0.f;
}

__global__ void loss_normalize_kernel(const float* __restrict__ loss_sum, const float* __restrict__ count,
                                      float count_host, float* __restrict__ inv_out, float* __restrict__ loss_out) {
  const float c = count ? *count : count_host;
  const float inv = 1.f / fmaxf(c, 1.f);
  if (inv_out) *inv_out = inv;
  if (loss_out) *loss_out = *loss_sum * inv;
}

__global__ void adamw_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ g, bf16* __restrict__ w, int64_t n, float lr, float b1, float b2,
                             float eps, float wd, float gscale, const float* __restrict__ gscale_dev, float bc1,
                             float bc2) {
  if (gscale_dev) gscale *= *gscale_dev;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i] * gscale;
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float mh = mi / bc1, vh = vi / bc2;
    float pi = p[i];
    pi -= lr * (mh / (sqrtf(vh) + eps)) + wd * pi;  // decoupled decay: wd is the per-step factor (R34)
    p[i] = pi;
    w[i] = __float2bfloat16_rn(pi);
  }
}

// the same update on 4 consecutive parameters per thread: 16-byte loads/stores of p, m, v, g and an
// 8-byte store of the bf16 weights (4x the bytes in flight per thread of the scalar loop)
__device__ __forceinline__ float adamw_one(float& p, float& m, float& v, float g, float lr, float b1, float b2,
                                           float eps, float wd, float gscale, float bc1, float bc2) {
  g *= gscale;
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  p -= lr * ((m / bc1) / (sqrtf(v / bc2) + eps)) + wd * p;
  return p;
}
__global__ void adamw4_kernel(float4* __restrict__ p, float4* __restrict__ m, float4* __restrict__ v,
                              const float4* __restrict__ g, uint2* __restrict__ w, int64_t n4, float lr, float b1,
                              float b2, float eps, float wd, float gscale, const float* __restrict__ gscale_dev,
                              float bc1, float bc2) {
  pdl_wait();
  pdl_trigger();
  if (gscale_dev) gscale *= *gscale_dev;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 pi = p[i], mi = m[i], vi = v[i];
    const float4 gi = g[i];
    adamw_one(pi.x, mi.x, vi.x, gi.x, lr, b1, b2, eps, wd, gscale, bc1, bc2);
    adamw_one(pi.y, mi.y, vi.y, gi.y, lr, b1, b2, eps, wd, gscale, bc1, bc2);
    adamw_one(pi.z, mi.z, vi.z, gi.z, lr, b1, b2, eps, wd, gscale, bc1, bc2);
    adamw_one(pi.w, mi.w, vi.w, gi.w, lr, b1, b2, eps, wd, gscale, bc1, bc2);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    const __nv_bfloat162 lo = __floats2bfloat162_rn(pi.x, pi.y), hi = __floats2bfloat162_rn(pi.z, pi.w);
    w[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
  }
}

inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// partial softmax statistics per row: one per (256-column tile, column half) of the decoder GEMM
inline int npart_of(int V) { return 2 * ((V + 255) / 256); }

struct HeadWs {
  bf16 *h, *tpre, *t, *u, *du;
  float *stats, *row_loss, *zlab;
  float2* part;
  bf16* dz;
  Det det;
  size_t bytes;
  HeadWs(char* base, int n, int H, int V, bool deterministic) {
    size_t o = 0;
    auto take = [&](size_t b) {
      char* p = base ? base + o : nullptr;
      o += al(b);
      return p;
    };
    h = (bf16*)take((size_t)n * H * 2);
    tpre = (bf16*)take((size_t)n * H * 2);
    t = (bf16*)take((size_t)n * H * 2);
    u = (bf16*)take((size_t)n * H * 2);
    du = (bf16*)take((size_t)n * H * 2);
    stats = (float*)take((size_t)n * 2 * 4);
    row_loss = (float*)take((size_t)n * 4);
    zlab = (float*)take((size_t)n * 4);
    part = (float2*)take((size_t)n * npart_of(V) * 8);
    dz = (bf16*)take((size_t)n * ((V + 7) & ~7) * 2);  // rows padded to 8 elements (any V, F3)
    if (deterministic) {
      det.part_floats = std::max(layernorm_bwd_det_floats(n, H), gemm_det_floats(V, H, n));
      det.part = (float*)take(det.part_floats * 4);
      det.sem_count = std::max(gemm_det_sems(V, H), gemm_det_sems(H, H));
      det.sem = (int*)take((size_t)det.sem_count * 4);
    }
    bytes = o;
  }
};

}  // namespace mb

extern "C" {

size_t mb_mlm_workspace_bytes(const mb_dims* d, int32_t n_masked) {
  if (!d) return 0;
  return mb::HeadWs(nullptr, std::max(n_masked, 1), d->hidden, d->vocab, (d->flags & MB_FLAG_DETERMINISTIC) != 0)
      .bytes;
}

mb_status mb_mlm_loss(const mb_dims* d, const mb_head_params* p, const mb_bf16* y, int32_t nnz,
                      const int32_t* masked_rows, const int32_t* labels, int32_t n_masked, float inv_norm,
                      float* loss_sum, float* lse, mb_bf16* dy_top, const mb_head_grads* g, void* ws, size_t ws_bytes,
                      mb_stream_t s_) {
  using namespace mb;
  if (!d || !p || !y || !masked_rows || !labels || !loss_sum || !lse || !ws) return MB_ERR_INVALID_ARG;
  const bool eval_only = !dy_top && !g;  // forward only: loss_sum and lse, no gradients (F4 evaluation)
  if (!eval_only && (!dy_top || !g)) return MB_ERR_INVALID_ARG;
  if (n_masked < 0 || nnz < 0) return MB_ERR_INVALID_ARG;
  if (n_masked > nnz) return MB_ERR_SHAPE;
  MB_REQUIRE_ARCH();
  const int H = d->hidden, V = d->vocab;
  if (V < 1 || H % 8) return MB_ERR_CONFIG;
  const int Vp = (V + 7) & ~7;  // dz row stride (P:174's 30522 is allowed; 30528 = 64 x 477 is the paper's choice)
  cudaStream_t s = reinterpret_cast<cudaStream_t>(s_);
  HeadWs w(reinterpret_cast<char*>(ws), std::max(n_masked, 1), H, V, (d->flags & MB_FLAG_DETERMINISTIC) != 0);
  if (ws_bytes < w.bytes) return MB_ERR_WORKSPACE;
  const Det* det = w.det ? &w.det : nullptr;
  bf16* dyt = reinterpret_cast<bf16*>(dy_top);
  if (n_masked == 0) {
    if (!eval_only && cudaMemsetAsync(dyt, 0, (size_t)nnz * H * 2, s) != cudaSuccess) return MB_ERR_CUDA;
    return MB_OK;
  }
  const int n = n_masked;
  if (det && cudaMemsetAsync(w.det.sem, 0, (size_t)w.det.sem_count * 4, s) != cudaSuccess) return MB_ERR_CUDA;
  auto B = [](const mb_bf16* q) { return reinterpret_cast<const bf16*>(q); };
  mb_status st;
#define TRY(x)                      \
  do {                              \
    if ((st = (x)) != MB_OK) return st; \
  } while (0)
  // forward: h = Y[rows]; t = GeLU(h W_t^T + b_t); u = LN_h(t); z = u E^T + b_dec
  TRY(gather_rows(B(y), masked_rows, n, H, w.h, s));
  {
    GemmArgs a;
    a.M = n, a.N = H, a.K = H, a.A = w.h, a.lda = H, a.B = B(p->w_t), a.ldb = H;
    a.ep.mode = E_GELU_AUX, a.ep.C = w.t, a.ep.ldc = H, a.ep.bias = B(p->b_t), a.ep.aux = w.tpre, a.ep.ldaux = H;
    TRY(gemm(a, s));
  }
  TRY(layernorm_fwd(w.t, B(p->ln_g), B(p->ln_b), n, H, d->ln_eps, w.u, w.stats, s));
  // z = u E^T + b_dec is never stored: the decoder GEMM's epilogue keeps an online (max, sum exp)
  // per row and tile and picks the label logit (E_LSE); a combine pass gives LSE and the row loss
  const int npart = npart_of(V);
  {
    GemmArgs a;
    a.M = n, a.N = V, a.K = H, a.A = w.u, a.lda = H, a.B = B(p->emb), a.ldb = H;
    a.ep.mode = E_LSE, a.ep.C = w.dz /* unused */, a.ep.ldc = Vp, a.ep.bias = B(p->b_dec);
    a.ep.labels = labels, a.ep.part = w.part, a.ep.zlab = w.zlab, a.ep.npart = npart;
    TRY(gemm(a, s));
  }
  ce_combine_kernel<<<(n + 7) / 8, 256, 0, s>>>(w.part, npart, w.zlab, n, lse, w.row_loss);
  MB_CHECK_LAUNCH();
  sum_kernel<<<1, 1024, 0, s>>>(w.row_loss, n, inv_norm, loss_sum);
  MB_CHECK_LAUNCH();
  if (eval_only) return MB_OK;
  // backward: recompute z tile by tile and emit dz = (softmax(z) - onehot(y)) * inv_norm (E_DZ)
  {
    GemmArgs a;
    a.M = n, a.N = V, a.K = H, a.A = w.u, a.lda = H, a.B = B(p->emb), a.ldb = H;
    a.ep.mode = E_DZ, a.ep.C = w.dz, a.ep.ldc = Vp, a.ep.bias = B(p->b_dec);
    a.ep.labels = labels, a.ep.lse = lse, a.ep.inv_norm = inv_norm;
    TRY(gemm(a, s));
  }
  {
    GemmArgs a;  // du = dz E   (E [V, H] = [K, N])
    a.M = n, a.N = H, a.K = V, a.A = w.dz, a.lda = Vp, a.B = B(p->emb), a.ldb = H, a.b_t = true;
    a.ep.mode = E_BF16, a.ep.C = w.du, a.ep.ldc = H;
    TRY(gemm(a, s));
  }
  {
    GemmArgs a;  // dE += dz^T u
    a.M = V, a.N = H, a.K = n, a.A = w.dz, a.lda = Vp, a.a_t = true, a.B = w.u, a.ldb = H, a.b_t = true;
    a.ep.mode = E_F32_ACC, a.ep.C = g->emb, a.ep.ldc = H;
    a.ep.dbias = g->b_dec;  // db_dec = column sums of dz, from the A tiles of this GEMM
    a.det = det;
    TRY(gemm(a, s));
  }
  // LN_h backward fused with the GeLU' of the transform: du -> dt_pre (in place); db_t = sum dt_pre
  TRY(layernorm_bwd(w.du, w.t, w.stats, B(p->ln_g), n, H, w.tpre, w.du, g->ln_g, g->ln_b, g->b_t, s, nullptr, nullptr,
                    det));
  {
    GemmArgs a;  // dh = dt_pre W_t  (W_t [H_out, H_in] = [K, N]) -> reuse t
    a.M = n, a.N = H, a.K = H, a.A = w.du, a.lda = H, a.B = B(p->w_t), a.ldb = H, a.b_t = true;
    a.ep.mode = E_BF16, a.ep.C = w.t, a.ep.ldc = H;
    TRY(gemm(a, s));
  }
  {
    GemmArgs a;  // dW_t += dt_pre^T h
    a.M = H, a.N = H, a.K = n, a.A = w.du, a.lda = H, a.a_t = true, a.B = w.h, a.ldb = H, a.b_t = true;
    a.ep.mode = E_F32_ACC, a.ep.C = g->w_t, a.ep.ldc = H;
    a.det = det;
    TRY(gemm(a, s));
  }
  TRY(scatter_rows(w.t, masked_rows, n, H, nnz, dyt, s));
#undef TRY
  return MB_OK;
}

mb_status mb_embed_forward(const mb_dims* d, const int32_t* ids, const int32_t* indices, int32_t nnz,
                           const mb_bf16* emb, const mb_bf16* type_emb, const mb_bf16* ln_g, const mb_bf16* ln_b,
                           mb_bf16* x0, float* stats, mb_stream_t s) {
  if (!d || !ids || !indices || !emb || !type_emb || !ln_g || !ln_b || !x0 || !stats || nnz < 0)
    return MB_ERR_INVALID_ARG;
  if (d->hidden % 8 || d->hidden > 1024 || d->vocab < 1) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  mb::EmbedSrc e;
  e.ids = ids, e.indices = indices, e.emb = reinterpret_cast<const bf16*>(emb);
  e.type_emb = reinterpret_cast<const bf16*>(type_emb);
  e.vocab = d->vocab;
  return mb::embed_ln_fwd(e, reinterpret_cast<const bf16*>(ln_g), reinterpret_cast<const bf16*>(ln_b), nnz, d->hidden,
                          d->ln_eps, reinterpret_cast<bf16*>(x0), stats, reinterpret_cast<cudaStream_t>(s));
}

size_t mb_embed_workspace_bytes(const mb_dims* d, int32_t nnz) {
  if (!d || !(d->flags & MB_FLAG_DETERMINISTIC) || nnz <= 0) return 0;
  const size_t ln = (mb::layernorm_bwd_det_floats(nnz, d->hidden) * 4 + 255) & ~size_t(255);
  return ln + mb::embed_det_bytes(nnz, d->hidden);
}

mb_status mb_embed_backward(const mb_dims* d, const int32_t* ids, const int32_t* indices, int32_t nnz,
                            const mb_bf16* emb, const mb_bf16* type_emb, const mb_bf16* ln_g, const float* stats,
                            mb_bf16* dx0, float* d_emb, float* d_type_emb, float* d_ln_g, float* d_ln_b, void* ws,
                            size_t ws_bytes, mb_stream_t s) {
  if (!d || !ids || !indices || !emb || !type_emb || !ln_g || !stats || !dx0 || !d_emb || !d_type_emb || !d_ln_g ||
      !d_ln_b || nnz < 0)
    return MB_ERR_INVALID_ARG;
  if (d->hidden % 8 || d->hidden > 1024 || d->vocab < 1) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  if (ws_bytes < mb_embed_workspace_bytes(d, nnz) || (ws_bytes && !ws)) return MB_ERR_WORKSPACE;
  mb::EmbedSrc e;
  e.ids = ids, e.indices = indices, e.emb = reinterpret_cast<const bf16*>(emb);
  e.type_emb = reinterpret_cast<const bf16*>(type_emb), e.d_emb = d_emb;
  e.vocab = d->vocab;
  mb::Det det;
  if ((d->flags & MB_FLAG_DETERMINISTIC) && nnz > 0) {
    char* w = reinterpret_cast<char*>(ws);
    det.part_floats = mb::layernorm_bwd_det_floats(nnz, d->hidden);
    det.part = reinterpret_cast<float*>(w);
    w += (det.part_floats * 4 + 255) & ~size_t(255);
    e.dv_out = reinterpret_cast<float*>(w);
    e.keys = reinterpret_cast<unsigned long long*>(w + (((size_t)nnz * d->hidden * 4 + 255) & ~size_t(255)));
  }
  // d_type_emb[0] = sum over tokens of dv (every token has type 0, R17) == the LN "dsum"
  return mb::embed_ln_bwd(e, reinterpret_cast<const bf16*>(dx0), stats, reinterpret_cast<const bf16*>(ln_g), nnz,
                          d->hidden, d_ln_g, d_ln_b, d_type_emb, reinterpret_cast<cudaStream_t>(s),
                          det ? &det : nullptr);
}

mb_status mb_adamw_step_dev(float* master, float* m, float* v, const float* g, mb_bf16* w_bf16, int64_t n,
                            float lr, float beta1, float beta2, float eps, float weight_decay, float grad_scale,
                            const float* grad_scale_dev, int32_t step, mb_stream_t s) {
  if (!master || !m || !v || !g || !w_bf16 || n < 0 || step < 1) return MB_ERR_INVALID_ARG;
  if (n == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  const bool vec = ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(m) |
                     reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(g)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(w_bf16) & 7) == 0;
  int64_t done = 0;
  if (vec && n >= 4) {
    const int64_t n4 = n / 4;
    const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 8 * mb::num_sms());
    if (mb::launch_pdl(mb::adamw4_kernel, dim3(grid), dim3(256), 0, st, 1, reinterpret_cast<float4*>(master),
                       reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                       reinterpret_cast<const float4*>(g), reinterpret_cast<uint2*>(w_bf16), n4, lr, beta1, beta2,
                       eps, weight_decay, grad_scale, grad_scale_dev, bc1, bc2) != cudaSuccess)
      return MB_ERR_CUDA;
    MB_CHECK_LAUNCH();
    done = n4 * 4;
  }
  if (done == n) return MB_OK;
  const int64_t rest = n - done;
  const int grid = (int)std::min<int64_t>((rest + 255) / 256, 8 * mb::num_sms());
  mb::adamw_kernel<<<grid, 256, 0, st>>>(master + done, m + done, v + done, g + done,
                                         reinterpret_cast<bf16*>(w_bf16) + done, rest, lr, beta1, beta2, eps,
                                         weight_decay, grad_scale, grad_scale_dev, bc1, bc2);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_loss_normalize(const float* loss_sum, const float* count, float count_host, float* inv_out,
                            float* loss_out, mb_stream_t s) {
  if (!loss_sum || (!inv_out && !loss_out)) return MB_ERR_INVALID_ARG;
  MB_REQUIRE_ARCH();
  mb::loss_normalize_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(s)>>>(loss_sum, count, count_host, inv_out,
                                                                          loss_out);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

double mb_lr_schedule(int64_t step, int64_t total_steps, double lr_peak) {
  if (total_steps <= 0) return lr_peak;
  const double T = (double)total_steps;
  const double t = (double)std::min<int64_t>(std::max<int64_t>(step, 0), total_steps);
  const double w = 0.06 * T;  // warmup: the first 6 % of the steps
  if (t <= w) return w > 0 ? lr_peak * t / w : lr_peak;
  return lr_peak * (1.0 - 0.98 * (t - w) / (T - w));  // linear to 0.02 lr_peak at T
}

mb_status mb_zero_f32(float* p, int64_t n, mb_stream_t s) {
  if (n < 0 || (n > 0 && !p)) return MB_ERR_INVALID_ARG;
  if (n == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  const int64_t head = std::min<int64_t>(n, (int64_t)((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / 4);
  const int64_t n4 = (n - head) / 4;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, 4 * mb::num_sms()));
  mb::zero_f32_kernel<<<grid, 256, 0, st>>>(p, n, head, n4);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_adamw_step(float* master, float* m, float* v, const float* g, mb_bf16* w_bf16, int64_t n, float lr,
                        float beta1, float beta2, float eps, float weight_decay, float grad_scale, int32_t step,
                        mb_stream_t s) {
  return mb_adamw_step_dev(master, m, v, g, w_bf16, n, lr, beta1, beta2, eps, weight_decay, grad_scale, nullptr, step,
                           s);
}

}  // extern "C"
