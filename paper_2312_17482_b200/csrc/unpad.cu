// A1/A2 — unpadding ("concatenate all the examples from a minibatch into a single sequence of
// batch size 1"): mask -> cu_seqlens / indices / max_seqlen, the MLM selection scan,
// and bf16 row gather/scatter.  Integer work: bit-exact by construction.
#include "common.cuh"

namespace mb {
namespace {

constexpr int SCAN_THREADS = 1024;

// Block-wide inclusive scan of one int per thread (1024 threads); returns the inclusive value and
// the block total.
__device__ __forceinline__ int block_scan_incl(int v, int* s_warp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) s_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += s_warp[warp - 1];
  total = s_warp[31];
  __syncthreads();
  return v;
}

// one CTA: phase 1 row counts + prefix check (warp per row, ballot/popc over 32-wide chunks),
// phase 2 exclusive scan over rows, phase 3 indices by rank.
// token-id range check of one real position (A3 reads E_tok[id]): bit 1 of the row's status
__device__ __forceinline__ int id_bad(const int* ids, int vocab, size_t pos) {
  if (!ids) return 0;
  const int id = ids[pos];
  return (id < 0 || id >= vocab) ? 2 : 0;
}
__device__ __forceinline__ int status_of(int bad) {
  return (bad & 1) ? MB_ERR_MASK_LAYOUT : (bad & 2) ? MB_ERR_TOKEN_RANGE : MB_OK;
}

__global__ void __launch_bounds__(SCAN_THREADS) unpad_index_kernel(const int* __restrict__ mask,
                                                                   const int* __restrict__ ids, int vocab, int B, int L,
                                                                   int* __restrict__ cu, int* __restrict__ indices,
                                                                   int* __restrict__ meta) {
  __shared__ int s_warp[32];
  __shared__ int s_bad, s_max;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_bad = 0;
    s_max = 0;
  }
  __syncthreads();
  int my_max = 0, my_bad = 0;
  for (int b = warp; b < B; b += SCAN_THREADS / 32) {
    const int* row = mask + (size_t)b * L;
    int cnt = 0, tok = 0;
    for (int l0 = 0; l0 < L; l0 += 32) {
      const int l = l0 + lane;
      const bool on = l < L && row[l] != 0;
      if (on) tok |= id_bad(ids, vocab, (size_t)b * L + l);
      cnt += __popc(__ballot_sync(0xffffffffu, on));
    }
    // right-padded prefix <=> every position l < cnt is on (R6)
    int bad = 0;
    for (int l0 = 0; l0 < cnt; l0 += 32) {
      const int l = l0 + lane;
      if (l < cnt && row[l] == 0) bad = 1;
    }
    bad = __any_sync(0xffffffffu, bad) | (__any_sync(0xffffffffu, tok) ? 2 : 0);
    if (lane == 0) {
      cu[b + 1] = cnt;
      my_max = max(my_max, cnt);
      my_bad |= bad;
    }
  }
  if (lane == 0) {
    atomicMax(&s_max, my_max);
    if (my_bad) atomicOr(&s_bad, my_bad);
  }
  __syncthreads();
  // phase 2: scan cu[1..B] in chunks of 1024
  int carry = 0;
  for (int base = 0; base < B; base += SCAN_THREADS) {
    const int b = base + threadIdx.x;
    const int v = b < B ? cu[b + 1] : 0;
    int tot;
    const int inc = block_scan_incl(v, s_warp, tot);
    if (b < B) cu[b + 1] = carry + inc;
    carry += tot;
  }
  if (threadIdx.x == 0) cu[0] = 0;
  __syncthreads();
  // phase 3: indices (ascending flat positions of the ones, also for non-prefix rows)
  for (int b = warp; b < B; b += SCAN_THREADS / 32) {
    const int* row = mask + (size_t)b * L;
    int out = cu[b];
    for (int l0 = 0; l0 < L; l0 += 32) {
      const int l = l0 + lane;
      const bool on = l < L && row[l] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (on) indices[out + __popc(bal & ((1u << lane) - 1u))] = b * L + l;
      out += __popc(bal);
    }
  }
  if (threadIdx.x == 0) {
    meta[0] = carry;
    meta[1] = s_max;
    meta[2] = status_of(s_bad);
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) mlm_select_kernel(const int* __restrict__ labels,
                                                                  const int* __restrict__ indices, int capacity,
                                                                  int vocab, int* __restrict__ rows,
                                                                  int* __restrict__ out_labels, int* __restrict__ meta,
                                                                  float* __restrict__ count_accum) {
  __shared__ int s_warp[32];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const int nnz = min(meta[0], capacity);
  int carry = 0, bad = 0;
  for (int base = 0; base < nnz; base += SCAN_THREADS) {
    const int t = base + threadIdx.x;
    int lab = -100;
    if (t < nnz) lab = labels[indices[t]];
    const int f = lab != -100;
    int tot;
    const int inc = block_scan_incl(f, s_warp, tot);
    if (f) {
      rows[carry + inc - 1] = t;
      out_labels[carry + inc - 1] = lab;
      if (lab < 0 || lab >= vocab) bad = 1;
    }
    carry += tot;
  }
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    meta[3] = carry;
    if (s_bad) meta[2] = MB_ERR_LABEL_RANGE;
    if (count_accum) *count_accum += (float)carry;
  }
}

// ---- multi-CTA unpad: (1) per-row counts + prefix check, warp per row; (2) every CTA sums the
// counts of the rows before its own (a few hundred ints) and writes its rows' indices, while CTA 0
// also writes cu_seqlens and meta.  Two short launches instead of one latency-bound CTA.
constexpr int UP_ROWS = 8;  // rows (warps) per CTA
__global__ void __launch_bounds__(UP_ROWS * 32) unpad_count_kernel(const int* __restrict__ mask,
                                                                   const int* __restrict__ ids, int vocab, int B, int L,
                                                                   int* __restrict__ cnt, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * UP_ROWS + (threadIdx.x >> 5);
  if (b >= B) return;
  const int* row = mask + (size_t)b * L;
  int c = 0, tok = 0;
  for (int l0 = 0; l0 < L; l0 += 32) {
    const int l = l0 + lane;
    const bool on = l < L && row[l] != 0;
    if (on) tok |= id_bad(ids, vocab, (size_t)b * L + l);
    c += __popc(__ballot_sync(0xffffffffu, on));
  }
  int nb = 0;  // right-padded prefix <=> every position l < c is on (R6)
  for (int l0 = 0; l0 < c; l0 += 32) {
    const int l = l0 + lane;
    if (l < c && row[l] == 0) nb = 1;
  }
  nb = __any_sync(0xffffffffu, nb) | (__any_sync(0xffffffffu, tok) ? 2 : 0);
  if (lane == 0) {
    cnt[b] = c;
    bad[b] = nb;
  }
}

__global__ void __launch_bounds__(UP_ROWS * 32) unpad_write_kernel(const int* __restrict__ mask, int B, int L,
                                                                   const int* __restrict__ cnt,
                                                                   const int* __restrict__ bad, int* __restrict__ cu,
                                                                   int* __restrict__ indices, int* __restrict__ meta) {
  __shared__ int s_part[UP_ROWS * 32 / 32];
  __shared__ int s_row[UP_ROWS + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = blockIdx.x * UP_ROWS;
  // exclusive prefix of this CTA's first row: sum of cnt[0 .. b0)
  int part = 0;
  for (int i = threadIdx.x; i < b0; i += blockDim.x) part += cnt[i];
  part = warp_sum_i(part);
  if (lane == 0) s_part[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    int base = 0;
    for (int w = 0; w < UP_ROWS; ++w) base += s_part[w];
    s_row[0] = base;
    for (int r = 0; r < UP_ROWS; ++r) s_row[r + 1] = s_row[r] + (b0 + r < B ? cnt[b0 + r] : 0);
  }
  __syncthreads();
  const int b = b0 + warp;
  if (b < B) {
    const int* row = mask + (size_t)b * L;
    int out = s_row[warp];
    for (int l0 = 0; l0 < L; l0 += 32) {
      const int l = l0 + lane;
      const bool on = l < L && row[l] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (on) indices[out + __popc(bal & ((1u << lane) - 1u))] = b * L + l;
      out += __popc(bal);
    }
  }
  if (blockIdx.x == 0) {  // cu_seqlens, nnz, max_seqlen, status
    __shared__ int s_warp[32];
    __shared__ int s_max, s_bad;
    if (threadIdx.x == 0) {
      s_max = 0;
      s_bad = 0;
    }
    __syncthreads();
    int carry = 0;
    for (int base = 0; base < B; base += blockDim.x) {
      const int i = base + threadIdx.x;
      const int v = i < B ? cnt[i] : 0;
      if (i < B) {
        atomicMax(&s_max, v);
        if (bad[i]) atomicOr(&s_bad, bad[i]);
      }
      // block inclusive scan (blockDim.x = 256 = 8 warps)
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      if (lane == 31) s_warp[warp] = x;
      __syncthreads();
      int off = 0, tot = 0;
      for (int w = 0; w < UP_ROWS; ++w) {
        if (w < warp) off += s_warp[w];
        tot += s_warp[w];
      }
      if (i < B) cu[i + 1] = carry + off + x;
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      cu[0] = 0;
      meta[0] = carry;
      meta[1] = s_max;
      meta[2] = status_of(s_bad);
    }
  }
}

// ---- multi-CTA MLM selection: (1) per-block counts of labelled tokens, (2) each block's prefix from
// the counts before it, block scan, ordered writes; the last block writes meta[3]
constexpr int SEL_THREADS = 1024;
__global__ void __launch_bounds__(SEL_THREADS) sel_count_kernel(const int* __restrict__ labels,
                                                                const int* __restrict__ indices, int capacity,
                                                                const int* __restrict__ meta, int* __restrict__ cnt) {
  __shared__ int s_warp[32];
  const int nnz = min(meta[0], capacity);
  const int t = blockIdx.x * SEL_THREADS + threadIdx.x;
  const int f = (t < nnz && labels[indices[t]] != -100) ? 1 : 0;
  int tot;
  block_scan_incl(f, s_warp, tot);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SEL_THREADS) sel_write_kernel(const int* __restrict__ labels,
                                                                const int* __restrict__ indices, int capacity,
                                                                int vocab, const int* __restrict__ cnt,
                                                                int* __restrict__ rows, int* __restrict__ out_labels,
                                                                int* __restrict__ meta, float* __restrict__ count_accum) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int nnz = min(meta[0], capacity);
  if (threadIdx.x < 32) {
    int p = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += 32) p += cnt[i];
    p = warp_sum_i(p);
    if (threadIdx.x == 0) s_base = p;
  }
  const int t = blockIdx.x * SEL_THREADS + threadIdx.x;
  const int lab = t < nnz ? labels[indices[t]] : -100;
  const int f = lab != -100;
  int tot;
  const int inc = block_scan_incl(f, s_warp, tot);  // includes a __syncthreads after s_base is set
  const int base = s_base;
  if (f) {
    rows[base + inc - 1] = t;
    out_labels[base + inc - 1] = lab;
    if (lab < 0 || lab >= vocab) meta[2] = MB_ERR_LABEL_RANGE;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    meta[3] = base + tot;
    if (count_accum) *count_accum += (float)(base + tot);
  }
}

// warp per row, 16-byte vectors
__global__ void gather_rows_kernel(const uint4* __restrict__ src, const int* __restrict__ idx, int n, int vec,
                                   uint4* __restrict__ dst) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const uint4* s = src + (size_t)idx[row] * vec;
  uint4* d = dst + (size_t)row * vec;
  for (int i = lane; i < vec; i += 32) d[i] = s[i];
}
__global__ void scatter_rows_kernel(const uint4* __restrict__ src, const int* __restrict__ idx, int n, int vec,
                                    uint4* __restrict__ dst) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const uint4* s = src + (size_t)row * vec;
  uint4* d = dst + (size_t)idx[row] * vec;
  for (int i = lane; i < vec; i += 32) d[i] = s[i];
}

}  // namespace

mb_status gather_rows(const bf16* src, const int* idx, int n, int H, bf16* dst, cudaStream_t s) {
  if (n == 0) return MB_OK;
  const int vec = H / 8;
  gather_rows_kernel<<<(n + 7) / 8, 256, 0, s>>>(reinterpret_cast<const uint4*>(src), idx, n, vec,
                                                 reinterpret_cast<uint4*>(dst));
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status scatter_rows(const bf16* src, const int* idx, int n, int H, int rows, bf16* dst, cudaStream_t s) {
  if (cudaMemsetAsync(dst, 0, (size_t)rows * H * sizeof(bf16), s) != cudaSuccess) return MB_ERR_CUDA;
  if (n == 0) return MB_OK;
  const int vec = H / 8;
  scatter_rows_kernel<<<(n + 7) / 8, 256, 0, s>>>(reinterpret_cast<const uint4*>(src), idx, n, vec,
                                                  reinterpret_cast<uint4*>(dst));
  MB_CHECK_LAUNCH();
  return MB_OK;
}

}  // namespace mb

extern "C" {

size_t mb_unpad_workspace_bytes(int32_t B) { return B > 0 ? 2 * (size_t)B * sizeof(int) : 0; }

size_t mb_select_workspace_bytes(int32_t capacity) {
  return capacity > 0 ? (size_t)((capacity + mb::SEL_THREADS - 1) / mb::SEL_THREADS) * sizeof(int) : 0;
}

mb_status mb_unpad_index(const int32_t* mask, const int32_t* ids, int32_t vocab, int32_t B, int32_t L,
                         int32_t* cu_seqlens, int32_t* indices, int32_t* meta, void* ws, size_t ws_bytes,
                         mb_stream_t s) {
  if (!mask || !cu_seqlens || !indices || !meta) return MB_ERR_INVALID_ARG;
  if (B <= 0 || L <= 0 || B > 65536 || L > 65536) return MB_ERR_INVALID_ARG;
  if (ids && vocab < 1) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  if (!ws) {  // no workspace: the single-CTA kernel
    mb::unpad_index_kernel<<<1, mb::SCAN_THREADS, 0, st>>>(mask, ids, vocab, B, L, cu_seqlens, indices, meta);
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  if (ws_bytes < mb_unpad_workspace_bytes(B)) return MB_ERR_WORKSPACE;
  int* scr = reinterpret_cast<int*>(ws);  // [0, B): row counts, [B, 2B): row status bits
  const int grid = (B + mb::UP_ROWS - 1) / mb::UP_ROWS;
  mb::unpad_count_kernel<<<grid, mb::UP_ROWS * 32, 0, st>>>(mask, ids, vocab, B, L, scr, scr + B);
  MB_CHECK_LAUNCH();
  mb::unpad_write_kernel<<<grid, mb::UP_ROWS * 32, 0, st>>>(mask, B, L, scr, scr + B, cu_seqlens, indices, meta);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_mlm_select(const int32_t* labels, const int32_t* indices, int32_t capacity, int32_t vocab,
                        int32_t* masked_rows, int32_t* masked_labels, int32_t* meta, float* count_accum, void* ws,
                        size_t ws_bytes, mb_stream_t s) {
  if (!labels || !indices || !masked_rows || !masked_labels || !meta) return MB_ERR_INVALID_ARG;
  if (capacity < 0) return MB_ERR_INVALID_ARG;
  if (vocab < 1) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  const int blocks = (capacity + mb::SEL_THREADS - 1) / mb::SEL_THREADS;
  if (!ws || blocks < 1) {  // no workspace / empty: the single-CTA kernel
    mb::mlm_select_kernel<<<1, mb::SCAN_THREADS, 0, st>>>(labels, indices, capacity, vocab, masked_rows,
                                                         masked_labels, meta, count_accum);
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  if (ws_bytes < mb_select_workspace_bytes(capacity)) return MB_ERR_WORKSPACE;
  int* scr = reinterpret_cast<int*>(ws);  // per-block label counts
  mb::sel_count_kernel<<<blocks, mb::SEL_THREADS, 0, st>>>(labels, indices, capacity, meta, scr);
  MB_CHECK_LAUNCH();
  mb::sel_write_kernel<<<blocks, mb::SEL_THREADS, 0, st>>>(labels, indices, capacity, vocab, scr, masked_rows,
                                                          masked_labels, meta, count_accum);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

mb_status mb_gather_rows(const mb_bf16* src, const int32_t* idx, int32_t n, int32_t H, mb_bf16* dst, mb_stream_t s) {
  if (!src || !idx || !dst || n < 0 || H <= 0) return MB_ERR_INVALID_ARG;
  if (H % 8) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  return mb::gather_rows(reinterpret_cast<const bf16*>(src), idx, n, H, reinterpret_cast<bf16*>(dst),
                         reinterpret_cast<cudaStream_t>(s));
}

mb_status mb_scatter_rows(const mb_bf16* src, const int32_t* idx, int32_t n, int32_t H, int32_t rows, mb_bf16* dst,
                          mb_stream_t s) {
  if (!src || !idx || !dst || n < 0 || H <= 0 || rows < n) return MB_ERR_INVALID_ARG;
  if (H % 8) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  return mb::scatter_rows(reinterpret_cast<const bf16*>(src), idx, n, H, rows, reinterpret_cast<bf16*>(dst),
                          reinterpret_cast<cudaStream_t>(s));
}

}  // extern "C"
