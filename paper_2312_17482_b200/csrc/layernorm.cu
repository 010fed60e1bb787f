// A7 / A3 — bf16 LayerNorm forward/backward (LN "run in bfloat16 ... only 2-bytes are
// required per-element"), the fused embedding gather + LN (no position table), and the
// bias-gradient column sums.
//
// One warp per row, 16-byte (8 x bf16) vector loads, VPL vectors per lane held in registers,
// warp-shuffle reductions; statistics, gamma/beta arithmetic and all reductions in fp32 (R12); the
// output is rounded once to bf16.  Backward column sums (dgamma, dbeta, and the preceding linear's
// bias gradient sum dx) accumulate per warp in registers, reduce per CTA through shared memory and
// reach global fp32 with one atomic per column per CTA.
#include <algorithm>
#include "common.cuh"
#include "kernels.h"

namespace mb {
namespace {

constexpr int LN_THREADS = 256;
constexpr int LN_WARPS = LN_THREADS / 32;

struct RowSrc {
  const bf16* x;          // plain mode: x[row*H]
  const int* ids;         // embed mode: x = emb[ids[indices[row]]] + type_emb[0]
  const int* indices;
  const bf16* emb;
  const bf16* type_emb;
  int vocab;              // embed mode: ids are clamped to [0, vocab) (out-of-range ids are reported
                          // by mb_unpad_index as MB_ERR_TOKEN_RANGE; the clamp keeps every access in bounds)
  float* dv_out;          // embed backward, deterministic mode: dv rows [n, H] fp32 instead of the scatter-add
};

template <int VPL, bool EMBED>
__device__ __forceinline__ void load_row(const RowSrc& src, int row, int H, int lane, float* v, int& id) {
  const bf16* base;
  if (EMBED) {
    id = min(max(src.ids[src.indices[row]], 0), src.vocab - 1);
    base = src.emb + (size_t)id * H;
  } else {
    base = src.x + (size_t)row * H;
  }
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = (i * 32 + lane) * 8;
    if (c < H) {
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(base + c), v + i * 8);
      if (EMBED) {
        float t[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(src.type_emb + c), t);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i * 8 + j] += t[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[i * 8 + j] = 0.f;
    }
  }
}

// Persistent variant for the encoder LNs: each warp walks rows with a grid stride, keeps gamma and
// beta in registers and has the next row's loads in flight while it reduces the current one (twice
// the bytes in flight per SM of the one-row-per-warp launch).
constexpr int LNP_BLOCKS = 3;  // resident CTAs per SM of the persistent forward
template <int VPL>
__global__ void __launch_bounds__(LN_THREADS, LNP_BLOCKS) ln_fwd_persist_kernel(const bf16* __restrict__ x,
                                                                                const bf16* __restrict__ gamma,
                                                                                const bf16* __restrict__ beta, int n,
                                                                                int H, float eps,
                                                                                bf16* __restrict__ y,
                                                                                float* __restrict__ stats) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int step = gridDim.x * LN_WARPS;
  uint4 nx[VPL];
  int row = blockIdx.x * LN_WARPS + (threadIdx.x >> 5);
  auto fetch = [&](int r) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (i * 32 + lane) * 8;
      nx[i] = c < H ? ld_nc_v4(x + (size_t)r * H + c) : make_uint4(0, 0, 0, 0);
    }
  };
  if (row < n) fetch(row);
  const float inv_h = __frcp_rn((float)H);
  for (; row < n; row += step) {
    float v[VPL * 8];
#pragma unroll
    for (int i = 0; i < VPL; ++i) bf16x8_to_f32(nx[i], v + i * 8);
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
        *reinterpret_cast<uint4*>(y + (size_t)row * H + c) = f32_to_bf16x8(o);
      }
    }
    if (lane == 0) *reinterpret_cast<float2*>(stats + 2 * (size_t)row) = make_float2(mean, rstd);
  }
}

template <int VPL, bool EMBED>
__global__ void __launch_bounds__(LN_THREADS) ln_fwd_kernel(RowSrc src, const bf16* __restrict__ gamma,
                                                            const bf16* __restrict__ beta, int n, int H, float eps,
                                                            bf16* __restrict__ y, float* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * LN_WARPS + (threadIdx.x >> 5);
  if (row >= n) return;
  float v[VPL * 8];
  int id;
  load_row<VPL, EMBED>(src, row, H, lane, v, id);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL * 8; ++i) s += v[i];
  const float inv_h = __frcp_rn((float)H);
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
      float g[8], b[8], o[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + c), g);
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(beta + c), b);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[i * 8 + j] - mean) * rstd * g[j] + b[j];
      *reinterpret_cast<uint4*>(y + (size_t)row * H + c) = f32_to_bf16x8(o);
    }
  }
  if (lane == 0) *reinterpret_cast<float2*>(stats + 2 * (size_t)row) = make_float2(mean, rstd);
}

// Reduce one per-lane register vector (the same column layout in every warp) across the CTA and
// atomically add it to out[H].
template <int VPL>
__device__ __forceinline__ void cta_column_reduce(const float* acc, float* sbuf, int H, float* out, float* part,
                                                  int j3) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = (i * 32 + lane) * 8;
    if (c < H) {
#pragma unroll
      for (int j = 0; j < 8; ++j) sbuf[warp * H + c + j] = acc[i * 8 + j];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += LN_THREADS) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < LN_WARPS; ++w) t += sbuf[w * H + c];
    if (part) part[((size_t)blockIdx.x * 3 + j3) * H + c] = t;  // deterministic mode: ordered second pass
    else atomicAdd(out + c, t);
  }
}

template <int VPL, bool EMBED, bool GELU, bool DSUM, bool DROP = false>
__global__ void __launch_bounds__(LN_THREADS, VPL <= 3 ? 2 : 1)
    ln_bwd_kernel(RowSrc src, const bf16* __restrict__ dy, const float* __restrict__ stats,
                  const bf16* __restrict__ gamma, const bf16* __restrict__ gelu_pre, int n, int H, bf16* dx,
                  float* __restrict__ d_emb, float* __restrict__ dgamma, float* __restrict__ dbeta,
                  float* __restrict__ dsum, DropArgs drop, bf16* __restrict__ dxd, float* __restrict__ part) {
  // Register budget (2 CTAs x 8 warps per SM): per lane only x-hat and the three column
  // accumulators stay live; dy and gamma are re-read (L1 hits) in the second pass.
  extern __shared__ float sbuf[];
  const int lane = threadIdx.x & 31;
  const float inv_h = __frcp_rn((float)H);
  float acc_g[VPL * 8], acc_b[VPL * 8], acc_s[DSUM ? VPL * 8 : 1];
#pragma unroll
  for (int i = 0; i < VPL * 8; ++i) {
    acc_g[i] = acc_b[i] = 0.f;
    if (DSUM) acc_s[i] = 0.f;
  }
  for (int row = blockIdx.x * LN_WARPS + (threadIdx.x >> 5); row < n; row += gridDim.x * LN_WARPS) {
    float v[VPL * 8];
    int id = 0;
    load_row<VPL, EMBED>(src, row, H, lane, v, id);
    const float2 st = *reinterpret_cast<const float2*>(stats + 2 * (size_t)row);
    const bf16* dyr = dy + (size_t)row * H;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < H) {
        float d[8], gm[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(dyr + c), d);
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + c), gm);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = i * 8 + j;
          const float xh = (v[k] - st.x) * st.y;
          v[k] = xh;
          const float gg = d[j] * gm[j];
          acc_g[k] += d[j] * xh;
          acc_b[k] += d[j];
          s1 += gg;
          s2 += gg * xh;
        }
      }
    }
    s1 = warp_sum(s1) * inv_h;
    s2 = warp_sum(s2) * inv_h;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (i * 32 + lane) * 8;
      if (c < H) {
        float d[8], gm[8], o[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(dyr + c), d);
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + c), gm);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = st.y * (d[j] * gm[j] - s1 - v[i * 8 + j] * s2);
        if (GELU) {
          float p[8];
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(gelu_pre + (size_t)row * H + c), p);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] *= gelu_grad_f(p[j]);
        }
        if (DROP) {  // F2: dx is the residual-path gradient; dxd = dx * keep / (1 - p) feeds the projection
          *reinterpret_cast<uint4*>(dx + (size_t)row * H + c) = f32_to_bf16x8(o);
          dropout_apply8(drop, (uint32_t)row, (uint32_t)c, o);
        }
        if (DSUM) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc_s[i * 8 + j] += o[j];
        }
        if (DROP) {
          *reinterpret_cast<uint4*>(dxd + (size_t)row * H + c) = f32_to_bf16x8(o);
        } else if (EMBED) {
          float* dst = src.dv_out ? src.dv_out + (size_t)row * H + c : d_emb + (size_t)id * H + c;
          if (src.dv_out) {
            *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<float4*>(dst + 4) = make_float4(o[4], o[5], o[6], o[7]);
          } else {
            red_add_v4(dst, o[0], o[1], o[2], o[3]);
            red_add_v4(dst + 4, o[4], o[5], o[6], o[7]);
          }
        } else {
          *reinterpret_cast<uint4*>(dx + (size_t)row * H + c) = f32_to_bf16x8(o);
        }
      }
    }
  }
  cta_column_reduce<VPL>(acc_g, sbuf, H, dgamma, part, 0);
  cta_column_reduce<VPL>(acc_b, sbuf, H, dbeta, part, 1);
  if (DSUM) cta_column_reduce<VPL>(acc_s, sbuf, H, dsum, part, 2);
}

// out[c] += sum_r x[r, c]; thread = one 8-column vector, blockIdx.y = row chunk
__global__ void colsum_kernel(const bf16* __restrict__ x, int n, int C, int rows_per, float* __restrict__ out) {
  const int cv = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = cv * 8;
  if (c >= C) return;
  const int r0 = blockIdx.y * rows_per, r1 = min(n, r0 + rows_per);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = r0; r < r1; ++r) {
    float f[8];
    bf16x8_to_f32(ld_nc_v4(x + (size_t)r * C + c), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += f[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) atomicAdd(out + c + j, acc[j]);
}


// LN backward with W warps per row (H = 256 W): every lane owns exactly one 16-byte vector of the
// row, so the three column accumulators cost 24 registers and the SM runs at full occupancy (the
// one-warp-per-row variant needed ~128 registers).  Row sums combine across the W warps through
// shared memory (double-buffered by row parity, one named barrier per row).
constexpr int LNW_GROUPS = 8;  // row groups (rows in flight) per CTA (8: half the CTAs, reductions and atomics of 4)
// Embedding backward (A3): dE_tok[id] += dx0 for every token.  A few ids occur thousands of times
// per batch ([MASK] is ~80 % of the 30 % masked positions, [CLS]/[SEP] open/close every sequence), and
// fp32 atomics on one row serialise in its L2 slice.  Each CTA therefore owns a contiguous range of
// <= EMB_ROWS rows, finds the ids that repeat >= EMB_HOT_MIN times inside it, accumulates those rows
// in shared memory (EMB_HOT slots) and flushes each slot once; all other rows go straight to L2.
constexpr int EMB_ROWS = 256, EMB_HOT = 4, EMB_HOT_MIN = 3;

template <int W, bool EMBED, bool GELU, bool DSUM, bool DROP = false>
__global__ void __launch_bounds__(LNW_GROUPS * W * 32)
    ln_bwd_w_kernel(RowSrc src, const bf16* __restrict__ dy, const float* __restrict__ stats,
                    const bf16* __restrict__ gamma, const bf16* __restrict__ gelu_pre, int n, int H, bf16* dx,
                    float* __restrict__ d_emb, float* __restrict__ dgamma, float* __restrict__ dbeta,
                    float* __restrict__ dsum, DropArgs drop, bf16* __restrict__ dxd, float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[LNW_GROUPS][2][W][2];
  extern __shared__ float sbuf[];  // [LNW_GROUPS][H] for the final column reduction (+ EMBED: [EMB_HOT][H])
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rg = warp / W, w = warp - rg * W;
  const int c = (w * 32 + lane) * 8;  // this lane's 8 columns
  const float inv_h = __frcp_rn((float)H);
  // EMBED: contiguous row range, its ids staged in smem, repeated ids given a shared-memory slot
  __shared__ int sid[EMBED ? EMB_ROWS : 1];
  __shared__ int hot[EMB_HOT];
  float* hacc = sbuf + LNW_GROUPS * H;
  int r_begin = 0, r_end = n;
  if (EMBED) {
    const int per = (n + gridDim.x - 1) / gridDim.x;
    r_begin = min(n, blockIdx.x * per);
    r_end = min(n, r_begin + per);
    const int cnt = r_end - r_begin;
    if (threadIdx.x < EMB_HOT) hot[threadIdx.x] = -1;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      sid[i] = min(max(src.ids[src.indices[r_begin + i]], 0), src.vocab - 1);
    for (int i = threadIdx.x; i < EMB_HOT * H; i += blockDim.x) hacc[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const int id = sid[i];
      int m = 0, first = i;
      for (int j = 0; j < cnt; ++j) {
        const bool eq = sid[j] == id;
        m += eq;
        if (eq && j < first) first = j;
      }
      if (m >= EMB_HOT_MIN && first == i) {  // one inserter per distinct id
        for (int k = 0; k < EMB_HOT; ++k)
          if (atomicCAS(&hot[k], -1, id) == -1) break;
      }
    }
    __syncthreads();
  }
  int hid[EMB_HOT];
#pragma unroll
  for (int k = 0; k < EMB_HOT; ++k) hid[k] = EMBED ? hot[k] : -1;
  float gm[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + c), gm);
  float ag[8], ab[8], as[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) ag[j] = ab[j] = as[j] = 0.f;
  int par = 0;
  // one-row-ahead prefetch of x, dy, stats (doubles the bytes in flight per SM)
  const int step = EMBED ? LNW_GROUPS : gridDim.x * LNW_GROUPS;
  auto fetch = [&](int r, uint4& xv, uint4& dv, float2& sv, int& idv) {
    const bf16* base;
    if (EMBED) {
      idv = sid[r - r_begin];
      base = src.emb + (size_t)idv * H;
    } else {
      base = src.x + (size_t)r * H;
    }
    xv = *reinterpret_cast<const uint4*>(base + c);
    dv = *reinterpret_cast<const uint4*>(dy + (size_t)r * H + c);
    sv = *reinterpret_cast<const float2*>(stats + 2 * (size_t)r);
  };
  uint4 nx = make_uint4(0, 0, 0, 0), nd = make_uint4(0, 0, 0, 0);
  float2 nst = make_float2(0.f, 0.f);
  int nid = 0;
  int row = EMBED ? r_begin + rg : blockIdx.x * LNW_GROUPS + rg;
  if (row < r_end) fetch(row, nx, nd, nst, nid);
  for (; row < r_end; row += step, par ^= 1) {
    const uint4 cx = nx, cd = nd;
    const float2 st = nst;
    const int id = nid;
    if (row + step < r_end) fetch(row + step, nx, nd, nst, nid);
    float xh[8], d[8];
    bf16x8_to_f32(cx, xh);
    if (EMBED) {
      float t[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(src.type_emb + c), t);
#pragma unroll
      for (int j = 0; j < 8; ++j) xh[j] += t[j];
    }
    bf16x8_to_f32(cd, d);
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
    for (int j = 0; j < 8; ++j) o[j] = st.y * (d[j] * gm[j] - s1 - xh[j] * s2);
    if (GELU) {
      float p[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(gelu_pre + (size_t)row * H + c), p);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] *= gelu_grad_f(p[j]);
    }
    if (DROP) {  // F2: dx is the residual-path gradient; dxd = dx * keep / (1 - p) feeds the projection
      *reinterpret_cast<uint4*>(dx + (size_t)row * H + c) = f32_to_bf16x8(o);
      dropout_apply8(drop, (uint32_t)row, (uint32_t)c, o);
    }
    if (DSUM) {
#pragma unroll
      for (int j = 0; j < 8; ++j) as[j] += o[j];
    }
    if (DROP) {
      *reinterpret_cast<uint4*>(dxd + (size_t)row * H + c) = f32_to_bf16x8(o);
    } else if (EMBED && src.dv_out) {  // deterministic mode: rows out, summed per id in token order later
      float* dst = src.dv_out + (size_t)row * H + c;
      *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<float4*>(dst + 4) = make_float4(o[4], o[5], o[6], o[7]);
    } else if (EMBED) {
      int slot = -1;
#pragma unroll
      for (int k = 0; k < EMB_HOT; ++k)
        if (hid[k] == id) slot = k;
      if (slot >= 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) atomicAdd(hacc + slot * H + c + j, o[j]);
      } else {
        float* dst = d_emb + (size_t)id * H + c;
        red_add_v4(dst, o[0], o[1], o[2], o[3]);
        red_add_v4(dst + 4, o[4], o[5], o[6], o[7]);
      }
    } else {
      *reinterpret_cast<uint4*>(dx + (size_t)row * H + c) = f32_to_bf16x8(o);
    }
  }
  // column sums: reduce the row groups through smem, one atomic per column per CTA
  auto reduce = [&](const float* acc, float* out, int j3) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) sbuf[rg * H + c + j] = acc[j];
    __syncthreads();
    for (int cc = threadIdx.x; cc < H; cc += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int g = 0; g < LNW_GROUPS; ++g) t += sbuf[g * H + cc];
      if (part) part[((size_t)blockIdx.x * 3 + j3) * H + cc] = t;  // deterministic mode: ordered second pass
      else atomicAdd(out + cc, t);
    }
  };
  reduce(ag, dgamma, 0);
  reduce(ab, dbeta, 1);
  if (DSUM) reduce(as, dsum, 2);
  if (EMBED && !src.dv_out) {  // flush the shared-memory rows of the repeated ids (every warp wrote: barrier first)
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < EMB_HOT; ++k) {
      if (hid[k] < 0) continue;
      for (int cc = threadIdx.x * 4; cc < H; cc += blockDim.x * 4)
        red_add_v4(d_emb + (size_t)hid[k] * H + cc, hacc[k * H + cc], hacc[k * H + cc + 1], hacc[k * H + cc + 2],
                   hacc[k * H + cc + 3]);
    }
  }
}

// deterministic mode: the per-CTA column partials [grid][3][H] are summed in CTA order afterwards
mb_status ln_det_finish(const Det* det, int grid, int H, float* dg, float* db, float* dsum, cudaStream_t s) {
  if (!det || !*det) return MB_OK;
  mb_status st;
  if ((st = ordered_sum(det->part, grid, 3 * (int64_t)H, H, dg, s)) != MB_OK) return st;
  if ((st = ordered_sum(det->part + H, grid, 3 * (int64_t)H, H, db, s)) != MB_OK) return st;
  if (dsum) return ordered_sum(det->part + 2 * H, grid, 3 * (int64_t)H, H, dsum, s);
  return MB_OK;
}

template <int W, bool EMBED>
mb_status ln_bwd_w_launch(const RowSrc& src, const bf16* dy, const float* stats, const bf16* gamma,
                          const bf16* gelu_pre, int n, int H, bf16* dx, float* d_emb, float* dg, float* db,
                          float* dsum, cudaStream_t s, const DropArgs& drop, bf16* dxd, const Det* det) {
  const int threads = LNW_GROUPS * W * 32;
  const int smem = (LNW_GROUPS + (EMBED ? EMB_HOT : 0)) * H * sizeof(float);
  const int blocks_per_sm = std::max(1, 2048 / threads);
  int grid = std::max(1, std::min((n + LNW_GROUPS - 1) / LNW_GROUPS, blocks_per_sm * num_sms()));
  if (EMBED) {
    grid = std::max(grid, (n + EMB_ROWS - 1) / EMB_ROWS);  // <= EMB_ROWS rows per CTA
    static bool attr = false;  // H = 1024: 48 KB dynamic + static smem exceeds the default window
    if (!attr) {
      if (cudaFuncSetAttribute(ln_bwd_w_kernel<W, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem) != cudaSuccess ||
          cudaFuncSetAttribute(ln_bwd_w_kernel<W, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               smem) != cudaSuccess)
        return MB_ERR_CUDA;
      attr = true;
    }
  }
  float* part = det && *det ? det->part : nullptr;
  if (part && det->part_floats < (size_t)grid * 3 * H) return MB_ERR_WORKSPACE;
#define LNW_GO(G, D)                                                                                           \
  ok = launch_pdl(ln_bwd_w_kernel<W, EMBED, G, D>, dim3(grid), dim3(threads), smem, s, 1, src, dy, stats, gamma, \
                  gelu_pre, n, H, dx, d_emb, dg, db, dsum, drop, dxd, part) == cudaSuccess
  bool ok = true;
  if (!EMBED && drop.thr) {
    if (gelu_pre || !dsum || !dxd) return MB_ERR_INVALID_ARG;
    ok = launch_pdl(ln_bwd_w_kernel<W, false, false, true, true>, dim3(grid), dim3(threads), smem, s, 1, src, dy, stats,
                    gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, drop, dxd, part) == cudaSuccess;
  } else if (gelu_pre && dsum) LNW_GO(true, true);
  else if (gelu_pre) LNW_GO(true, false);
  else if (dsum) LNW_GO(false, true);
  else LNW_GO(false, false);
#undef LNW_GO
  if (!ok) return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  return ln_det_finish(det, grid, H, dg, db, dsum, s);
}

template <bool EMBED>
mb_status ln_fwd_dispatch(const RowSrc& src, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                          float* stats, cudaStream_t s) {
  if (n == 0) return MB_OK;
  const int grid = (n + LN_WARPS - 1) / LN_WARPS;
  const int vpl = (H / 8 + 31) / 32;
  if (!EMBED && (vpl == 3 || vpl == 4) && n >= 4096) {
    const int pgrid = std::min(grid, LNP_BLOCKS * num_sms());  // one resident wave, rows strided
    bool ok;
    if (vpl == 3)
      ok = launch_pdl(ln_fwd_persist_kernel<3>, dim3(pgrid), dim3(LN_THREADS), 0, s, 1, src.x, gamma, beta, n, H, eps,
                      y, stats) == cudaSuccess;
    else
      ok = launch_pdl(ln_fwd_persist_kernel<4>, dim3(pgrid), dim3(LN_THREADS), 0, s, 1, src.x, gamma, beta, n, H, eps,
                      y, stats) == cudaSuccess;
    if (!ok) return MB_ERR_CUDA;
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  switch (vpl) {
    case 1: ln_fwd_kernel<1, EMBED><<<grid, LN_THREADS, 0, s>>>(src, gamma, beta, n, H, eps, y, stats); break;
    case 2: ln_fwd_kernel<2, EMBED><<<grid, LN_THREADS, 0, s>>>(src, gamma, beta, n, H, eps, y, stats); break;
    case 3: ln_fwd_kernel<3, EMBED><<<grid, LN_THREADS, 0, s>>>(src, gamma, beta, n, H, eps, y, stats); break;
    case 4: ln_fwd_kernel<4, EMBED><<<grid, LN_THREADS, 0, s>>>(src, gamma, beta, n, H, eps, y, stats); break;
    default: return MB_ERR_CONFIG;
  }
  MB_CHECK_LAUNCH();
  return MB_OK;
}

template <int VPL, bool EMBED>
mb_status ln_bwd_launch(const RowSrc& src, const bf16* dy, const float* stats, const bf16* gamma,
                        const bf16* gelu_pre, int n, int H, bf16* dx, float* d_emb, float* dg, float* db,
                        float* dsum, cudaStream_t s, const DropArgs& drop, bf16* dxd, const Det* det) {
  const int smem = LN_WARPS * H * sizeof(float);
  const int grid = std::max(1, std::min((n + LN_WARPS - 1) / LN_WARPS, (VPL <= 3 ? 2 : 1) * num_sms()));
  float* part = det && *det ? det->part : nullptr;
  if (part && det->part_floats < (size_t)grid * 3 * H) return MB_ERR_WORKSPACE;
  if (!EMBED && drop.thr) {
    if (gelu_pre || !dsum || !dxd) return MB_ERR_INVALID_ARG;
    ln_bwd_kernel<VPL, false, false, true, true><<<grid, LN_THREADS, smem, s>>>(src, dy, stats, gamma, gelu_pre, n,
                                                                                H, dx, d_emb, dg, db, dsum, drop,
                                                                                dxd, part);
  } else if (gelu_pre && dsum)
    ln_bwd_kernel<VPL, EMBED, true, true><<<grid, LN_THREADS, smem, s>>>(src, dy, stats, gamma, gelu_pre, n, H, dx,
                                                                          d_emb, dg, db, dsum, drop, dxd, part);
  else if (gelu_pre)
    ln_bwd_kernel<VPL, EMBED, true, false><<<grid, LN_THREADS, smem, s>>>(src, dy, stats, gamma, gelu_pre, n, H, dx,
                                                                           d_emb, dg, db, dsum, drop, dxd, part);
  else if (dsum)
    ln_bwd_kernel<VPL, EMBED, false, true><<<grid, LN_THREADS, smem, s>>>(src, dy, stats, gamma, gelu_pre, n, H,
                                                                           dx, d_emb, dg, db, dsum, drop, dxd, part);
  else
    ln_bwd_kernel<VPL, EMBED, false, false><<<grid, LN_THREADS, smem, s>>>(src, dy, stats, gamma, gelu_pre, n, H,
                                                                            dx, d_emb, dg, db, dsum, drop, dxd, part);
  MB_CHECK_LAUNCH();
  return ln_det_finish(det, grid, H, dg, db, dsum, s);
}

template <bool EMBED>
mb_status ln_bwd_dispatch(const RowSrc& src, const bf16* dy, const float* stats, const bf16* gamma,
                          const bf16* gelu_pre, int n, int H, bf16* dx, float* d_emb, float* dg, float* db,
                          float* dsum, cudaStream_t s, const DropArgs& drop = DropArgs(), bf16* dxd = nullptr,
                          const Det* det = nullptr) {
  if (n == 0) return MB_OK;
  if (H == 768) return ln_bwd_w_launch<3, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
  if (H == 1024) return ln_bwd_w_launch<4, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
  if (H == 512) return ln_bwd_w_launch<2, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
  if (H == 256) return ln_bwd_w_launch<1, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
  switch ((H / 8 + 31) / 32) {
    case 1: return ln_bwd_launch<1, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
    case 2: return ln_bwd_launch<2, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
    case 3: return ln_bwd_launch<3, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
    case 4: return ln_bwd_launch<4, EMBED>(src, dy, stats, gamma, gelu_pre, n, H, dx, d_emb, dg, db, dsum, s, drop, dxd, det);
  }
  return MB_ERR_CONFIG;
}

}  // namespace

mb_status layernorm_fwd(const bf16* x, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                        float* stats, cudaStream_t s) {
  RowSrc src{x, nullptr, nullptr, nullptr, nullptr, 0, nullptr};
  return ln_fwd_dispatch<false>(src, gamma, beta, n, H, eps, y, stats, s);
}

mb_status layernorm_bwd(const bf16* dy, const bf16* x, const float* stats, const bf16* gamma, int n, int H,
                        const bf16* gelu_pre, bf16* dx, float* dgamma, float* dbeta, float* dsum, cudaStream_t s,
                        const DropArgs* drop, bf16* dxd, const Det* det) {
  RowSrc src{x, nullptr, nullptr, nullptr, nullptr, 0, nullptr};
  const DropArgs none;
  return ln_bwd_dispatch<false>(src, dy, stats, gamma, gelu_pre, n, H, dx, nullptr, dgamma, dbeta, dsum, s,
                                drop ? *drop : none, dxd, det);
}

size_t layernorm_bwd_det_floats(int n, int H) {
  // bound on every LN-backward grid (ln_bwd_w_launch: <= 8 CTAs/SM or n / EMB_ROWS; ln_bwd_launch: 2/SM)
  const size_t grid = (size_t)8 * num_sms() + (size_t)n / EMB_ROWS + 8;
  return grid * 3 * (size_t)H;
}

mb_status embed_ln_fwd(const EmbedSrc& e, const bf16* gamma, const bf16* beta, int n, int H, float eps, bf16* y,
                       float* stats, cudaStream_t s) {
  RowSrc src{nullptr, e.ids, e.indices, e.emb, e.type_emb, e.vocab, nullptr};
  return ln_fwd_dispatch<true>(src, gamma, beta, n, H, eps, y, stats, s);
}

mb_status embed_ln_bwd(const EmbedSrc& e, const bf16* dy, const float* stats, const bf16* gamma, int n, int H,
                       float* dgamma, float* dbeta, float* dsum, cudaStream_t s, const Det* det) {
  const bool dm = det && *det;
  if (dm) MB_REQUIRE(e.dv_out && e.keys, MB_ERR_WORKSPACE);
  RowSrc src{nullptr, e.ids, e.indices, e.emb, e.type_emb, e.vocab, dm ? e.dv_out : nullptr};
  mb_status st = ln_bwd_dispatch<true>(src, dy, stats, gamma, nullptr, n, H, nullptr, e.d_emb, dgamma, dbeta, dsum,
                                       s, DropArgs(), nullptr, det);
  if (st != MB_OK || !dm) return st;
  // deterministic scatter-add: sort the (id, token) pairs, then each id's rows are summed in token order
  return embed_scatter_det(e.dv_out, e.ids, e.indices, n, H, e.vocab, e.keys, e.d_emb, s);
}

mb_status colsum(const bf16* x, int n, int C, float* out, cudaStream_t s) {
  if (n == 0 || C == 0) return MB_OK;
  if (C % 8) return MB_ERR_CONFIG;
  const int cvec = C / 8;
  const int bx = (cvec + 127) / 128;
  const int target = 4 * num_sms();
  int by = std::max(1, std::min((target + bx - 1) / bx, (n + 63) / 64));
  const int rows_per = (n + by - 1) / by;
  by = (n + rows_per - 1) / rows_per;
  colsum_kernel<<<dim3(bx, by), 128, 0, s>>>(x, n, C, rows_per, out);
  MB_CHECK_LAUNCH();
  return MB_OK;
}

}  // namespace mb

extern "C" {

mb_status mb_layernorm_forward(const mb_bf16* x, const mb_bf16* gamma, const mb_bf16* beta, int32_t n, int32_t H,
                               float eps, mb_bf16* y, float* stats, mb_stream_t s) {
  if (!x || !gamma || !beta || !y || !stats || n < 0 || H <= 0) return MB_ERR_INVALID_ARG;
  if (H % 8 || H > 1024) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  return mb::layernorm_fwd(reinterpret_cast<const bf16*>(x), reinterpret_cast<const bf16*>(gamma),
                           reinterpret_cast<const bf16*>(beta), n, H, eps, reinterpret_cast<bf16*>(y), stats,
                           reinterpret_cast<cudaStream_t>(s));
}

mb_status mb_layernorm_backward(const mb_bf16* dy, const mb_bf16* x, const float* stats, const mb_bf16* gamma,
                                int32_t n, int32_t H, const mb_bf16* gelu_pre, mb_bf16* dx, float* dgamma,
                                float* dbeta, float* dsum, mb_stream_t s) {
  if (!dy || !x || !stats || !gamma || !dx || !dgamma || !dbeta || n < 0 || H <= 0) return MB_ERR_INVALID_ARG;
  if (H % 8 || H > 1024) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  return mb::layernorm_bwd(reinterpret_cast<const bf16*>(dy), reinterpret_cast<const bf16*>(x), stats,
                           reinterpret_cast<const bf16*>(gamma), n, H, reinterpret_cast<const bf16*>(gelu_pre),
                           reinterpret_cast<bf16*>(dx), dgamma, dbeta, dsum, reinterpret_cast<cudaStream_t>(s));
}

mb_status mb_colsum(const mb_bf16* x, int32_t n, int32_t C, float* out, mb_stream_t s) {
  if (!x || !out || n < 0 || C < 0) return MB_ERR_INVALID_ARG;
  MB_REQUIRE_ARCH();
  return mb::colsum(reinterpret_cast<const bf16*>(x), n, C, out, reinterpret_cast<cudaStream_t>(s));
}

}  // extern "C"
