// F3 — baselines for the paper's throughput ablations, built from the same kernel
// designs as the hot path so that each ablation isolates one of the paper's choices:
//   * fp32 LayerNorm (the paper's bf16 LN halves the bytes of a bandwidth-bound op): the
//     persistent forward and the W-warps-per-row backward of layernorm.cu with fp32 activations;
//   * the naive (unfused) GLU ("the extra elementwise multiplication" and different
//     GEMM calls): two separate projections through mb_gemm plus these elementwise GeGLU kernels,
//     saving the pre-activations as autograd would.
// Padded-vs-varlen attention and vocab 30522-vs-30528 need no extra kernels (bench inputs only).
#include <algorithm>
#include "common.cuh"
#include "kernels.h"

namespace mb {
namespace {

constexpr int AB_THREADS = 256, AB_WARPS = AB_THREADS / 32;

__device__ __forceinline__ void ld8_f32(const float* p, float* v) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void st8_f32(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

// y = LN(x) with fp32 x / y (gamma, beta bf16 as in the model); persistent, next row prefetched
template <int VPL>
__global__ void __launch_bounds__(AB_THREADS, 2) ln_fwd_f32_kernel(const float* __restrict__ x,
                                                                   const bf16* __restrict__ gamma,
                                                                   const bf16* __restrict__ beta, int n, int H,
                                                                   float eps, float* __restrict__ y,
                                                                   float* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int step = gridDim.x * AB_WARPS;
  float nx[VPL * 8];
  int row = blockIdx.x * AB_WARPS + (threadIdx.x >> 5);
  auto fetch = [&](int r) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < H) ld8_f32(x + (size_t)r * H + c, nx + i * 8);
      else
#pragma unroll
        for (int j = 0; j < 8; ++j) nx[i * 8 + j] = 0.f;
    }
  };
  if (row < n) fetch(row);
  const float inv_h = __frcp_rn((float)H);
  for (; row < n; row += step) {
    float v[VPL * 8];
#pragma unroll
    for (int i = 0; i < VPL * 8; ++i) v[i] = nx[i];
    if (row + step < n) fetch(row + step);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPL * 8; ++i) s += v[i];
    const float mean = warp_sum(s) * inv_h;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < H) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = v[i * 8 + j] - mean;
          q += d * d;
        }
      }
    }
    const float rstd = rsqrtf(warp_sum(q) * inv_h + eps);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < H) {
        float g[8], bt[8], o[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + c), g);
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(beta + c), bt);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[i * 8 + j] - mean) * rstd * g[j] + bt[j];
        st8_f32(y + (size_t)row * H + c, o);
      }
    }
    if (lane == 0) *reinterpret_cast<float2*>(stats + 2 * (size_t)row) = make_float2(mean, rstd);
  }
}

// dx = LN backward with fp32 dy / x / dx; W warps per row, column sums dgamma, dbeta, dsum (= the
// preceding linear's bias gradient) per CTA through smem, one atomic per column per CTA
constexpr int ABW_GROUPS = 4;
template <int W>
__global__ void __launch_bounds__(ABW_GROUPS * W * 32)
    ln_bwd_f32_kernel(const float* __restrict__ x, const float* __restrict__ dy, const float* __restrict__ stats,
                      const bf16* __restrict__ gamma, int n, int H, float* __restrict__ dx,
                      float* __restrict__ dgamma, float* __restrict__ dbeta, float* __restrict__ dsum) {
  __shared__ float red[ABW_GROUPS][2][W][2];
  extern __shared__ float sbuf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rg = warp / W, w = warp - rg * W;
  const int c = (w * 32 + lane) * 8;
  const float inv_h = __frcp_rn((float)H);
  float gm[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + c), gm);
  float ag[8], ab[8], as[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) ag[j] = ab[j] = as[j] = 0.f;
  int par = 0;
  const int step = gridDim.x * ABW_GROUPS;
  for (int row = blockIdx.x * ABW_GROUPS + rg; row < n; row += step, par ^= 1) {
    float xh[8], d[8];
    ld8_f32(x + (size_t)row * H + c, xh);
    ld8_f32(dy + (size_t)row * H + c, d);
    const float2 st = *reinterpret_cast<const float2*>(stats + 2 * (size_t)row);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      xh[j] = (xh[j] - st.x) * st.y;
      const float g = d[j] * gm[j];
      ag[j] += d[j] * xh[j];
      ab[j] += d[j];
      s1 += g;
      s2 += g * xh[j];
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (W > 1) {
      if (lane == 0) {
        red[rg][par][w][0] = s1;
        red[rg][par][w][1] = s2;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + rg), "r"(W * 32) : "memory");
      s1 = 0.f;
      s2 = 0.f;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        s1 += red[rg][par][k][0];
        s2 += red[rg][par][k][1];
      }
    }
    s1 *= inv_h;
    s2 *= inv_h;
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      o[j] = st.y * (d[j] * gm[j] - s1 - xh[j] * s2);
      as[j] += o[j];
    }
    st8_f32(dx + (size_t)row * H + c, o);
  }
  auto reduce = [&](const float* acc, float* out) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) sbuf[rg * H + c + j] = acc[j];
    __syncthreads();
    for (int cc = threadIdx.x; cc < H; cc += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int g = 0; g < ABW_GROUPS; ++g) t += sbuf[g * H + cc];
      atomicAdd(out + cc, t);
    }
  };
  reduce(ag, dgamma);
  reduce(ab, dbeta);
  if (dsum) reduce(as, dsum);
}

// naive GLU, elementwise part: Z = GeLU(Ua) * Ug  (exact-erf GeLU, R7; bf16 in / out)
__global__ void geglu_ew_fwd_kernel(const bf16* __restrict__ ua, const bf16* __restrict__ ug, int64_t n8,
                                    bf16* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float a[8], g[8], o[8];
    bf16x8_to_f32(ld_nc_v4(ua + 8 * i), a);
    bf16x8_to_f32(ld_nc_v4(ug + 8 * i), g);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = gelu_f(a[e]) * g[e];
    *reinterpret_cast<uint4*>(z + 8 * i) = f32_to_bf16x8(o);
  }
}
// dUa = dZ * Ug * GeLU'(Ua), dUg = dZ * GeLU(Ua)
__global__ void geglu_ew_bwd_kernel(const bf16* __restrict__ dz, const bf16* __restrict__ ua,
                                    const bf16* __restrict__ ug, int64_t n8, bf16* __restrict__ dua,
                                    bf16* __restrict__ dug) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float d[8], a[8], g[8], oa[8], og[8];
    bf16x8_to_f32(ld_nc_v4(dz + 8 * i), d);
    bf16x8_to_f32(ld_nc_v4(ua + 8 * i), a);
    bf16x8_to_f32(ld_nc_v4(ug + 8 * i), g);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float cdf, pdf;
      norm_cdf_pdf(a[e], cdf, pdf);
      oa[e] = d[e] * g[e] * (cdf + a[e] * pdf);
      og[e] = d[e] * a[e] * cdf;
    }
    *reinterpret_cast<uint4*>(dua + 8 * i) = f32_to_bf16x8(oa);
    *reinterpret_cast<uint4*>(dug + 8 * i) = f32_to_bf16x8(og);
  }
}

}  // namespace
}  // namespace mb

extern "C" {

mb_status mb_layernorm_forward_f32(const float* x, const mb_bf16* gamma, const mb_bf16* beta, int32_t n, int32_t H,
                                   float eps, float* y, float* stats, mb_stream_t s_) {
  using namespace mb;
  if (!x || !gamma || !beta || !y || !stats || n < 0 || H <= 0) return MB_ERR_INVALID_ARG;
  if (H % 8 || H > 1024) return MB_ERR_CONFIG;
  if (n == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(s_);
  const int grid = std::max(1, std::min((n + AB_WARPS - 1) / AB_WARPS, 2 * num_sms()));
  const auto g = reinterpret_cast<const bf16*>(gamma);
  const auto b = reinterpret_cast<const bf16*>(beta);
  switch ((H / 8 + 31) / 32) {
    case 1: ln_fwd_f32_kernel<1><<<grid, AB_THREADS, 0, s>>>(x, g, b, n, H, eps, y, stats); break;
    case 2: ln_fwd_f32_kernel<2><<<grid, AB_THREADS, 0, s>>>(x, g, b, n, H, eps, y, stats); break;
    case 3: ln_fwd_f32_kernel<3><<<grid, AB_THREADS, 0, s>>>(x, g, b, n, H, eps, y, stats); break;
    default: ln_fwd_f32_kernel<4><<<grid, AB_THREADS, 0, s>>>(x, g, b, n, H, eps, y, stats); break;
  }
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_layernorm_backward_f32(const float* dy, const float* x, const float* stats, const mb_bf16* gamma,
                                    int32_t n, int32_t H, float* dx, float* dgamma, float* dbeta, float* dsum,
                                    mb_stream_t s_) {
  using namespace mb;
  if (!dy || !x || !stats || !gamma || !dx || !dgamma || !dbeta || n < 0 || H <= 0) return MB_ERR_INVALID_ARG;
  if (H % 256 || H > 1024) return MB_ERR_CONFIG;
  if (n == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(s_);
  const auto g = reinterpret_cast<const bf16*>(gamma);
  const int W = H / 256, threads = ABW_GROUPS * W * 32;
  const int smem = ABW_GROUPS * H * sizeof(float);
  const int grid = std::max(1, std::min((n + ABW_GROUPS - 1) / ABW_GROUPS, std::max(1, 2048 / threads) * num_sms()));
  switch (W) {
    case 1: ln_bwd_f32_kernel<1><<<grid, threads, smem, s>>>(x, dy, stats, g, n, H, dx, dgamma, dbeta, dsum); break;
    case 2: ln_bwd_f32_kernel<2><<<grid, threads, smem, s>>>(x, dy, stats, g, n, H, dx, dgamma, dbeta, dsum); break;
    case 3: ln_bwd_f32_kernel<3><<<grid, threads, smem, s>>>(x, dy, stats, g, n, H, dx, dgamma, dbeta, dsum); break;
    default: ln_bwd_f32_kernel<4><<<grid, threads, smem, s>>>(x, dy, stats, g, n, H, dx, dgamma, dbeta, dsum); break;
  }
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_geglu_naive_forward(const mb_bf16* ua, const mb_bf16* ug, int64_t count, mb_bf16* z, mb_stream_t s_) {
  using namespace mb;
  if (!ua || !ug || !z || count < 0) return MB_ERR_INVALID_ARG;
  if (count % 8) return MB_ERR_CONFIG;
  if (count == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  const int64_t n8 = count / 8;
  const int grid = (int)std::min<int64_t>((n8 + 255) / 256, 8 * num_sms());
  geglu_ew_fwd_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(s_)>>>(
      reinterpret_cast<const bf16*>(ua), reinterpret_cast<const bf16*>(ug), n8, reinterpret_cast<bf16*>(z));
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_geglu_naive_backward(const mb_bf16* dz, const mb_bf16* ua, const mb_bf16* ug, int64_t count,
                                  mb_bf16* dua, mb_bf16* dug, mb_stream_t s_) {
  using namespace mb;
  if (!dz || !ua || !ug || !dua || !dug || count < 0) return MB_ERR_INVALID_ARG;
  if (count % 8) return MB_ERR_CONFIG;
  if (count == 0) return MB_OK;
  MB_REQUIRE_ARCH();
  const int64_t n8 = count / 8;
  const int grid = (int)std::min<int64_t>((n8 + 255) / 256, 8 * num_sms());
  geglu_ew_bwd_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(s_)>>>(
      reinterpret_cast<const bf16*>(dz), reinterpret_cast<const bf16*>(ua), reinterpret_cast<const bf16*>(ug), n8,
      reinterpret_cast<bf16*>(dua), reinterpret_cast<bf16*>(dug));
  MB_CHECK_LAUNCH();
  return MB_OK;
}

}  // extern "C"
