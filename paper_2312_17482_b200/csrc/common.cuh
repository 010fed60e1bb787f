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

// exact-erf GeLU (reading R7) and its derivative Phi(x) + x phi(x)
__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  const float pdf = 0.3989422804014327f * __expf(-0.5f * x * x);
  return cdf + x * pdf;
}

int num_sms();  // cached per device (host)
void count_launch();  // host-side counter of kernel launches (mb_launch_count)
// optional timing probe around one kernel site (mb_probe_set): records caller-provided CUDA events
enum ProbeSite { PROBE_NONE = 0, PROBE_GEGLU_FWD = 1, PROBE_ATTN_FWD = 2, PROBE_ATTN_BWD = 3, PROBE_LN_FWD = 4 };
void probe_begin(int site, cudaStream_t s);
void probe_end(int site, cudaStream_t s);

}  // namespace mb
