// Host runtime pieces of the C ABI: status strings, version, device attribute cache, TMA maps,
// ALiBi slopes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include "common.cuh"
#include "tma.h"

namespace mb {

static int g_sms[64];
static std::once_flag g_sms_once[64];

bool pdl_enabled() {
  static const bool on = std::getenv("MB_NO_PDL") == nullptr;
  return on;
}

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  std::call_once(g_sms_once[dev], [dev] {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 148;
    // MB_SM_CARVEOUT=k: the persistent grids leave k SMs idle (kept even for the CTA pairs), where a
    // concurrent NCCL bucket reduction runs without waiting for a kernel boundary (data parallelism)
    const char* c = std::getenv("MB_SM_CARVEOUT");
    const int k = c ? std::atoi(c) : 0;
    if (k > 0 && k < n - 2) n = (n - k) & ~1;
    g_sms[dev] = n;
  });
  return g_sms[dev];
}

// MB_ERR_ARCH: the SASS in this library is sm_100a only (B200).  Cached per device.
static int g_arch[64];
static std::once_flag g_arch_once[64];
bool arch_ok() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::call_once(g_arch_once[dev], [dev] {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    g_arch[dev] = (major == 10 && minor == 0) ? 1 : 0;
  });
  return g_arch[dev] == 1;
}

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct Probe {
  int site = PROBE_NONE;
  cudaEvent_t* events = nullptr;
  int capacity = 0;
  int* count = nullptr;
};
static Probe g_probe;
void probe_begin(int site, cudaStream_t s) {
  if (site != g_probe.site || !g_probe.events) return;
  const int i = *g_probe.count;
  if (2 * i + 1 < g_probe.capacity && cudaEventRecord(g_probe.events[2 * i], s) != cudaSuccess)
    cudaGetLastError();  // a bad probe must never poison the compute path's launch checks
}
void probe_end(int site, cudaStream_t s) {
  if (site != g_probe.site || !g_probe.events) return;
  const int i = *g_probe.count;
  if (2 * i + 1 < g_probe.capacity) {
    if (cudaEventRecord(g_probe.events[2 * i + 1], s) == cudaSuccess) *g_probe.count = i + 1;
    else cudaGetLastError();
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                       uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                   : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                         : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_f32_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace mb

extern "C" {

const char* mb_status_string(int s) {
  switch (s) {
    case MB_OK: return "MB_OK";
    case MB_ERR_INVALID_ARG: return "MB_ERR_INVALID_ARG";
    case MB_ERR_CONFIG: return "MB_ERR_CONFIG";
    case MB_ERR_SHAPE: return "MB_ERR_SHAPE";
    case MB_ERR_MASK_LAYOUT: return "MB_ERR_MASK_LAYOUT";
    case MB_ERR_LABEL_RANGE: return "MB_ERR_LABEL_RANGE";
    case MB_ERR_WORKSPACE: return "MB_ERR_WORKSPACE";
    case MB_ERR_ARCH: return "MB_ERR_ARCH";
    case MB_ERR_CUDA: return "MB_ERR_CUDA";
    case MB_ERR_TOKEN_RANGE: return "MB_ERR_TOKEN_RANGE";
  }
  return "MB_ERR_UNKNOWN";
}

const char* mb_version(void) { return "mosaicbert-b200 0.1 (sm_100a)"; }

unsigned long long mb_launch_count(void) { return mb::g_launches.load(); }

mb_status mb_probe_set(int32_t site, void* events, int32_t capacity, int32_t* count) {
  if (site != 0 && (!events || !count || capacity < 2)) return MB_ERR_INVALID_ARG;
  mb::g_probe.site = site;
  mb::g_probe.events = reinterpret_cast<cudaEvent_t*>(events);
  mb::g_probe.capacity = capacity;
  mb::g_probe.count = count;
  return MB_OK;
}

// geometric sequence with ratio 2^(-8/n) starting at 2^(-8/n) (R3).  Computed in double
// and rounded once to float, so it is the correctly rounded fp32 value of the closed form.
mb_status mb_alibi_slopes(int32_t heads, float* out) {
  if (!out) return MB_ERR_INVALID_ARG;
  if (heads <= 0) return MB_ERR_CONFIG;
  for (int h = 0; h < heads; ++h) out[h] = (float)exp2(-8.0 * (double)(h + 1) / (double)heads);
  return MB_OK;
}

}  // extern "C"
