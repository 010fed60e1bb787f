// Deterministic fp32 reductions (SURVEY §8a E6 "split-K partials reduced deterministically", A7
// "per-CTA fp32 partials + a deterministic second pass"): the second passes of the deterministic
// mode.  Every partial is produced by exactly one CTA with plain stores; these kernels add them in a
// fixed order, so the result is bitwise identical from run to run (the default mode adds the same
// partials with fp32 atomics, whose order varies).
#include "common.cuh"
#include "kernels.h"

namespace mb {
namespace {

// out[c] += sum_p part[p * stride + c], p ascending; one thread per column
__global__ void ordered_sum_kernel(const float* __restrict__ part, int nparts, int64_t stride, int count,
                                   float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  float t = 0.f;
  for (int p = 0; p < nparts; ++p) t += part[(int64_t)p * stride + c];
  out[c] += t;
}

constexpr int CS_ROWS = 512;  // rows per chunk of the deterministic column sum

// part[chunk * C + c] = sum of rows [chunk * CS_ROWS, +CS_ROWS) of column c (rows ascending)
__global__ void colsum_chunk_kernel(const bf16* __restrict__ x, int64_t ldx, int n, int C, float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= C) return;
  const int r0 = blockIdx.y * CS_ROWS, r1 = min(n, r0 + CS_ROWS);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = r0; r < r1; ++r) {
    float f[8];
    bf16x8_to_f32(ld_nc_v4(x + (int64_t)r * ldx + c), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += f[j];
  }
  float* dst = part + (int64_t)blockIdx.y * C + c;
#pragma unroll
  for (int j = 0; j < 8; ++j) dst[j] = acc[j];
}

// ---- deterministic embedding scatter (A3 backward, MB_FLAG_DETERMINISTIC) --------------------------
// keys[t] = (id << 32) | t for t < n, all-ones padding up to the power of two N2
__global__ void emb_keys_kernel(const int* __restrict__ ids, const int* __restrict__ indices, int n, int vocab, int N2,
                                unsigned long long* __restrict__ keys) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N2) return;
  if (t < n) {
    const int id = min(max(ids[indices[t]], 0), vocab - 1);
    keys[t] = ((unsigned long long)(unsigned)id << 32) | (unsigned)t;
  } else {
    keys[t] = ~0ull;
  }
}

constexpr int BS_ELEMS = 2048;  // elements per CTA in the shared-memory bitonic stages (1024 threads)

__device__ __forceinline__ void cmp_swap(unsigned long long& a, unsigned long long& b, bool asc) {
  if ((a > b) == asc) {
    const unsigned long long t = a;
    a = b;
    b = t;
  }
}

// all stages (k, j) with j < BS_ELEMS of merge sizes k in [k_lo, k_hi] on this CTA's 2048 elements
__global__ void __launch_bounds__(1024) bitonic_local_kernel(unsigned long long* __restrict__ keys, int k_lo, int k_hi) {
  __shared__ unsigned long long sk[BS_ELEMS];
  const int base = blockIdx.x * BS_ELEMS;
  for (int i = threadIdx.x; i < BS_ELEMS; i += blockDim.x) sk[i] = keys[base + i];
  __syncthreads();
  for (int k = k_lo; k <= k_hi; k <<= 1) {
    for (int j = min(k >> 1, BS_ELEMS >> 1); j > 0; j >>= 1) {
      const int i = 2 * threadIdx.x - (threadIdx.x & (j - 1));  // lower index of this thread's pair
      const int g = base + i;                                   // global index (direction from k)
      cmp_swap(sk[i], sk[i + j], (g & k) == 0);
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < BS_ELEMS; i += blockDim.x) keys[base + i] = sk[i];
}

// one global stage (k, j), j >= BS_ELEMS
__global__ void bitonic_global_kernel(unsigned long long* __restrict__ keys, int k, int j) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = 2 * t - (t & (j - 1));
  unsigned long long a = keys[i], b = keys[i + j];
  const unsigned long long a0 = a;
  cmp_swap(a, b, (i & k) == 0);
  if (a != a0) {
    keys[i] = a;
    keys[i + j] = b;
  }
}

// one CTA per sorted position p that starts an id's run: d_emb[id] += its rows in ascending token
// order (four interleaved partial sums, combined in a fixed order); the only writer of that row
__global__ void emb_segment_kernel(const unsigned long long* __restrict__ keys, int n, const float* __restrict__ dv,
                                   int H, float* __restrict__ d_emb) {
  const int p = blockIdx.x;
  const unsigned id = (unsigned)(keys[p] >> 32);
  if (p > 0 && (unsigned)(keys[p - 1] >> 32) == id) return;
  const int c = threadIdx.x * 4;
  if (c >= H) return;
  float4 acc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  int q = p;
  for (; q + 3 < n && (unsigned)(keys[q + 3] >> 32) == id; q += 4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned t = (unsigned)(keys[q + k] & 0xffffffffu);
      const float4 v = __ldcs(reinterpret_cast<const float4*>(dv + (size_t)t * H + c));
      acc[k].x += v.x, acc[k].y += v.y, acc[k].z += v.z, acc[k].w += v.w;
    }
  }
  for (; q < n && (unsigned)(keys[q] >> 32) == id; ++q) {
    const unsigned t = (unsigned)(keys[q] & 0xffffffffu);
    const float4 v = __ldcs(reinterpret_cast<const float4*>(dv + (size_t)t * H + c));
    acc[0].x += v.x, acc[0].y += v.y, acc[0].z += v.z, acc[0].w += v.w;
  }
  float4* dst = reinterpret_cast<float4*>(d_emb + (size_t)id * H + c);
  float4 o = *dst;
  o.x += (acc[0].x + acc[1].x) + (acc[2].x + acc[3].x);
  o.y += (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y);
  o.z += (acc[0].z + acc[1].z) + (acc[2].z + acc[3].z);
  o.w += (acc[0].w + acc[1].w) + (acc[2].w + acc[3].w);
  *dst = o;
}

int pow2_at_least(int n) {
  int p = BS_ELEMS;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace

size_t embed_det_bytes(int n, int H) {
  const size_t dv = ((size_t)n * H * sizeof(float) + 255) & ~size_t(255);
  return dv + (size_t)pow2_at_least(n) * sizeof(unsigned long long);
}

mb_status embed_scatter_det(const float* dv, const int* ids, const int* indices, int n, int H, int vocab,
                            unsigned long long* keys, float* d_emb, cudaStream_t s) {
  if (n <= 0) return MB_OK;
  if (H % 4 || H > 4096) return MB_ERR_CONFIG;
  const int N2 = pow2_at_least(n);
  if (launch_pdl(emb_keys_kernel, dim3((N2 + 255) / 256), dim3(256), 0, s, 1, ids, indices, n, vocab, N2, keys) !=
      cudaSuccess)
    return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  const int blocks = N2 / BS_ELEMS;
  bitonic_local_kernel<<<blocks, 1024, 0, s>>>(keys, 2, BS_ELEMS);
  MB_CHECK_LAUNCH();
  for (int k = 2 * BS_ELEMS; k <= N2; k <<= 1) {
    for (int j = k >> 1; j >= BS_ELEMS; j >>= 1) {
      bitonic_global_kernel<<<N2 / 2 / 256, 256, 0, s>>>(keys, k, j);
      MB_CHECK_LAUNCH();
    }
    bitonic_local_kernel<<<blocks, 1024, 0, s>>>(keys, k, k);
    MB_CHECK_LAUNCH();
  }
  emb_segment_kernel<<<n, (H / 4 + 31) / 32 * 32, 0, s>>>(keys, n, dv, H, d_emb);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status ordered_sum(const float* part, int nparts, int64_t stride, int count, float* out, cudaStream_t s) {
  if (count <= 0 || nparts <= 0) return MB_OK;
  if (launch_pdl(ordered_sum_kernel, dim3((count + 255) / 256), dim3(256), 0, s, 1, part, nparts, stride, count,
                 out) != cudaSuccess)
    return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  return MB_OK;
}

size_t colsum_det_floats(int n, int C) { return (size_t)((n + CS_ROWS - 1) / CS_ROWS) * (size_t)C; }

mb_status colsum_det(const bf16* x, int64_t ldx, int n, int C, float* out, float* part, cudaStream_t s) {
  if (n <= 0 || C <= 0) return MB_OK;
  if (C % 8 || ldx % 8) return MB_ERR_CONFIG;
  const int chunks = (n + CS_ROWS - 1) / CS_ROWS;
  const int cv = C / 8;
  if (launch_pdl(colsum_chunk_kernel, dim3((cv + 127) / 128, chunks), dim3(128), 0, s, 1, x, ldx, n, C, part) !=
      cudaSuccess)
    return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  return ordered_sum(part, chunks, C, C, out, s);
}

}  // namespace mb
