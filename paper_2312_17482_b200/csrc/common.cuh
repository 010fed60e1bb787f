// Shared device/host helpers for the MosaicBERT sm_100a kernels (no method arithmetic here).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../../include/mosaicbert.h"

typedef __nv_bfloat16 bf16;
typedef __nv_bfloat162 bf162;

#define MB_CHECK_LAUNCH()                                   \
  do {                                                      \
    mb::count_launch();                                     \
    cudaError_t e__ = cudaGetLastError();                   \
    if (e__ != cudaSuccess) return MB_ERR_CUDA;             \
  } while (0)

// every entry point that touches the device: MB_ERR_ARCH on anything but sm_100 (B200)
#define MB_REQUIRE_ARCH()                     \
  do {                                        \
    if (!mb::arch_ok()) return MB_ERR_ARCH;   \
  } while (0)

#define MB_REQUIRE(cond, code) \
  do {                         \
    if (!(cond)) return (code);\
  } while (0)

namespace mb {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 8 bf16 <-> 8 float through one 16-byte vector
__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const bf162* h = reinterpret_cast<const bf162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 u;
  bf162* h = reinterpret_cast<bf162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  bf162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Standard-normal cdf Phi(x) and pdf phi(x) sharing one exponential: Phi(x) = 0.5 (1 + erf(x/sqrt2))
// with erf from Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, far below bf16 resolution):
//   erf(z) = 1 - t (a1 + t (a2 + t (a3 + t (a4 + t a5)))) e^{-z^2},  t = 1 / (1 + p z),  z >= 0,
// and e^{-z^2} = e^{-x^2/2} is exactly the exponential of phi.  GeLU(x) = x Phi(x) is the exact-erf
// GeLU (reading R7) to fp32 accuracy; GeLU'(x) = Phi(x) + x phi(x).
__device__ __forceinline__ void norm_cdf_pdf(float x, float& cdf, float& pdf) {
  const float e = exp2f(-0.72134752044448170f * x * x);  // e^{-x^2/2}
  const float t = __fdividef(1.0f, fmaf(0.2316418882663604f, fabsf(x), 1.0f));  // p / sqrt2
  float q = fmaf(t, 0.5307027145f, -0.7265760135f);  // halved a5, a4 (0.5 folded in)
  q = fmaf(t, q, 0.7107068705f);
  q = fmaf(t, q, -0.1422483680f);
  q = fmaf(t, q, 0.1274147960f);
  q = q * t * e;  // = 0.5 (1 - erf(|x|/sqrt2))
  cdf = x >= 0.f ? 1.0f - q : q;
  pdf = 0.3989422804014327f * e;
}
// norm_cdf_pdf for two values on the paired fp32 pipe (sm_100 FFMA2/FMUL2), same A&S 7.1.26 form:
// e = 2^{-x^2 log2(e)/2}, t = 1/(1 + p|x|/sqrt2), q = 0.5 t poly(t) e, cdf = 0.5 + sgn(x)(0.5 - q).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void norm_cdf_pdf2(float2 x, float2& cdf, float2& pdf) {
  const float2 xx = __fmul2_rn(x, x);
  const float2 ea = __fmul2_rn(xx, make_float2(-0.72134752044448170f, -0.72134752044448170f));
  const float2 e = make_float2(ex2_approx(ea.x), ex2_approx(ea.y));
  const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
  const float2 den = __ffma2_rn(ax, make_float2(0.2316418882663604f, 0.2316418882663604f), make_float2(1.f, 1.f));
  const float2 t = make_float2(rcp_approx(den.x), rcp_approx(den.y));
  float2 q = __ffma2_rn(t, make_float2(0.5307027145f, 0.5307027145f), make_float2(-0.7265760135f, -0.7265760135f));
  q = __ffma2_rn(t, q, make_float2(0.7107068705f, 0.7107068705f));
  q = __ffma2_rn(t, q, make_float2(-0.1422483680f, -0.1422483680f));
  q = __ffma2_rn(t, q, make_float2(0.1274147960f, 0.1274147960f));
  q = __fmul2_rn(__fmul2_rn(q, t), e);  // = 0.5 (1 - erf(|x|/sqrt2))
  const float2 h = __ffma2_rn(q, make_float2(-1.f, -1.f), make_float2(0.5f, 0.5f));
  const float2 sg = make_float2(copysignf(1.f, x.x), copysignf(1.f, x.y));
  cdf = __ffma2_rn(sg, h, make_float2(0.5f, 0.5f));
  pdf = __fmul2_rn(e, make_float2(0.3989422804014327f, 0.3989422804014327f));
}
// ---- F2 dropout (reading R32): Philox-4x32-10 (Salmon et al., SC'11) keyed by the seed,
// counter (f >> 3, packed row t, 2*stream + site, 0); 16-bit field (f & 1) of word (f & 7) >> 1 is
// the uniform of feature f; kept iff >= thr = round(65536 p).
struct DropArgs {
  uint32_t key0 = 0, key1 = 0;  // seed mod 2^32, seed >> 32
  uint32_t site = 0;            // 2 * stream + {0: attention out-proj, 1: FFN down-proj}
  uint32_t thr = 0;             // 0 = dropout off
  float scale = 1.f;            // 1 / (1 - p)
};
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}
// keep bits of features [f0, f0 + 8) (f0 % 8 == 0) of packed row t: bit j <-> feature f0 + j
__device__ __forceinline__ uint32_t dropout_keep8(const DropArgs& d, uint32_t t, uint32_t f0) {
  const uint4 w = philox4x32_10(make_uint4(f0 >> 3, t, d.site, 0u), d.key0, d.key1);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) bits |= (uint32_t)(((ws[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) >= d.thr) << j;
  return bits;
}
// v[0..8) of features f0.. of row t -> v * keep * scale
__device__ __forceinline__ void dropout_apply8(const DropArgs& d, uint32_t t, uint32_t f0, float* v) {
  const uint32_t bits = dropout_keep8(d, t, f0);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = ((bits >> j) & 1u) ? v[j] * d.scale : 0.f;
}

__device__ __forceinline__ float gelu_f(float x) {
  float c, p;
  norm_cdf_pdf(x, c, p);
  return x * c;
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  float c, p;
  norm_cdf_pdf(x, c, p);
  return c + x * p;
}

// Programmatic dependent launch (PDL).  A kernel launched through launch_pdl() may become resident
// while its predecessor in the stream is still draining (its prologue — barrier init, TMEM alloc,
// tensor-map prefetch — overlaps the predecessor's tail).  It must call pdl_wait() before it
// touches global memory that earlier kernels write; pdl_trigger() then lets its own successor
// start launching.  Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();  // host: true unless the environment sets MB_NO_PDL (A/B measurements)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

int num_sms();  // cached per device (host)
bool arch_ok();  // host: the current device is sm_100 (the only SASS this library carries)
void count_launch();  // host-side counter of kernel launches (mb_launch_count)
// optional timing probe around one kernel site (mb_probe_set): records caller-provided CUDA events
enum ProbeSite { PROBE_NONE = 0, PROBE_GEGLU_FWD = 1, PROBE_ATTN_FWD = 2, PROBE_ATTN_BWD = 3, PROBE_LN_FWD = 4 };
void probe_begin(int site, cudaStream_t s);
void probe_end(int site, cudaStream_t s);

}  // namespace mb
