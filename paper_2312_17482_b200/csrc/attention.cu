// A5 / A10 — variable-length FlashAttention with in-kernel ALiBi (Eq. 1; FlashAttention
// P:120) on the unpadded token stream, forward and backward, on tcgen05 tensor cores.
//
//   s_ij = q_i . k_j / sqrt(d) - m_h |i - j|      (i, j = positions inside one sequence; R2, R4)
//
// All kernels are persistent and warp-specialised: TMA producer / MMA issuer lanes plus 8 softmax
// warps (two threads per 128-row tile row, 64 keys each).  Q/K/V/dO tiles come straight out of the
// packed buffers by TMA (128-byte swizzle, rows past the sequence are masked, rows past nnz read as
// 0); S = Q K^T, dP = dO V^T, O = P V, dV = P^T dO, dK = dS^T Q, dQ = dS K all run as tcgen05.mma
// kind::f16 with fp32 accumulators in TMEM.  A thread reads its half-row of S from TMEM
// (tcgen05.ld), adds the ALiBi bias computed from the two positions (never materialised), does the
// exp2-domain softmax in fp32 on the paired fp32 pipe, and writes P / dS as bf16 into shared memory
// in the same swizzled layout the next MMA consumes (K-major for P V and dS K, MN-major for the
// transposed P^T dO and dS^T Q — the same bytes serve both views).  Outputs leave by per-warp TMA
// stores of 64B-swizzled [32 x 32] blocks.
//   l <= 128 (C1/C2/C3/C5): one unit = (sequence, head), single-pass softmax.
//   128 < l <= 2048 (C4, F4): forward units = (query tile, head, sequence) with the online softmax
//   over key tiles; backward units = (key tile, head, sequence) over query tiles, dQ reduced in fp32.
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma.h"

namespace mb {
namespace {

constexpr int TILE = 128;
constexpr int DT = 64;  // head-dim tile in shared memory (d = 32 uses half of it; the rest is ignored)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
constexpr int TILE_BYTES = TILE * DT * 2;  // 16 KB
constexpr int P_BYTES = TILE * TILE * 2;   // 32 KB

// byte offset of element (row r, column c) of a [128 x 128] bf16 tile stored as two 64-column
// 128B-swizzled atoms (K-major for the row index as M), c multiple of 8
__device__ __forceinline__ uint32_t p_off(int r, int c) {
  return (uint32_t)((c >> 6) * (TILE * 128) + (r >> 3) * 1024 + (r & 7) * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4));
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ------------------------------------------------------------------------------------------
// Short-sequence path (l <= 128: every workload of BASELINE configs 1, 2, 3, 5): one (sequence,
// head) unit = one Q tile and one K/V tile, single-pass softmax (no rescaling).  Persistent CTAs of
// 8 warps: warp w reads TMEM lane quarter (w & 3) and column half (w >> 2), so two threads share a
// query row and exchange its max / sum through shared memory.  The next unit's TMA loads are issued
// as soon as the MMAs that read the current tiles have completed, overlapping the output epilogue.
// ------------------------------------------------------------------------------------------
constexpr int SH_THREADS = 256;
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

__device__ __forceinline__ int unit_len(const int* cu, int heads, int u) {
  const int b = u / heads;
  return cu[b + 1] - cu[b];
}
__device__ __forceinline__ int next_unit(const int* cu, int heads, int total, int u) {
  for (u += gridDim.x; u < total; u += gridDim.x)
    if (unit_len(cu, heads, u) > 0) return u;
  return total;
}

// Forward scores of this thread's 64 keys [64 ch, 64 ch + 64) of query row r, in the exp2 domain:
// x_j = S_rj log2e / sqrt(d) - m_h log2e |r - j| (-inf past the sequence when MASK); returns max_j.
template <bool MASK>
__device__ __forceinline__ float fwd_scores(float (&x)[64], int r, int ch, int len, float sc2, float sl2,
                                           int qk_off = 0) {
  // query position - key position of this thread's first key = r + qk_off - 64 ch (qk_off = q0 - kv0);
  // keys at or past len (relative to the tile) are masked
  const float rc = (float)(r + qk_off - 64 * ch);
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 64; j += 2) {
    const float2 dd = __fadd2_rn(make_float2(rc, rc), make_float2(-(float)j, -(float)j - 1.f));
    const float2 t = __ffma2_rn(make_float2(fabsf(dd.x), fabsf(dd.y)), make_float2(-sl2, -sl2),
                                __fmul2_rn(make_float2(x[j], x[j + 1]), make_float2(sc2, sc2)));
    x[j] = t.x;
    x[j + 1] = t.y;
    if (MASK) {
      x[j] = 64 * ch + j < len ? x[j] : -INFINITY;
      x[j + 1] = 64 * ch + j + 1 < len ? x[j + 1] : -INFINITY;
    }
    mx = fmaxf(mx, fmaxf(x[j], x[j + 1]));
  }
  return mx;
}

// Forward, software-pipelined: warp 8 (one lane) issues the TMA loads of units i+1, i+2 into two
// smem buffers and S(i+1) = Q K^T into the second TMEM S buffer while warps 0-7 run the softmax of
// unit i; then O(i) = P V into one of two TMEM O buffers.  The softmax warps read O(i) out only
// after the softmax of unit i+1, so the PV latency hides behind useful work (P is double-buffered
// in smem for that).  TMEM: S[0] [0,128), S[1] [128,256), O[0] [256,320), O[1] [320,384).
constexpr int SH_FWD_THREADS = SH_THREADS + 32;
constexpr int FWD_BUF_BYTES = 3 * TILE_BYTES;  // Q, K, V
constexpr int FWD_NBUF = 3;                    // Q/K/V buffers: loads run two units ahead
constexpr int SH_FWD_SMEM2 = FWD_NBUF * FWD_BUF_BYTES + 2 * P_BYTES + 1024 + 256;

__global__ void __launch_bounds__(SH_FWD_THREADS, 1) attn_fwd_short_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                                                                          const __grid_constant__ CUtensorMap tm_o,
                                                                          const int* __restrict__ cu, int batch,
                                                                          int heads, int d,
                                                                          const float* __restrict__ slopes,
                                                                          bf16* __restrict__ O,
                                                                          float* __restrict__ lse, int nnz) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bufs = smem;  // FWD_NBUF x (Q, K, V)
  uint8_t* sP = smem + FWD_NBUF * FWD_BUF_BYTES;  // 2 x P (unit i's P buffer also stages O(i))
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * P_BYTES);
  uint64_t* load_full = bars;     // [FWD_NBUF]
  // one S barrier per TMEM S buffer: S(i+1) is committed before the softmax of unit i ends, so a
  // single barrier could run two phases ahead of a slow waiter (parity aliasing); same for O
  uint64_t* s_full = bars + 3;    // [2]
  // [2] by unit parity, 8 compute warps arrive per unit: S(i+1) is in TMEM before unit i's P is
  // complete, so a fast warp pair can arrive for unit i+1 while a slow pair is still on unit i; a
  // single barrier would count that arrival towards unit i's phase
  uint64_t* p_ready = bars + 5;
  uint64_t* o_full = bars + 7;    // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9);
  __shared__ float rmax[2 * 128], rsum[2 * 128];  // half-row max / sum exchange of the two row threads

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = heads * d;
  const int total = batch * heads;
  if (tid == 0) {
    sm100::tma_prefetch(&tm_qkv);
    sm100::tma_prefetch(&tm_o);
    for (int k = 0; k < FWD_NBUF; ++k) sm100::mbar_init(&load_full[k], 1);
    sm100::mbar_init(&s_full[0], 1);
    sm100::mbar_init(&s_full[1], 1);
    sm100::mbar_init(&p_ready[0], 8);
    sm100::mbar_init(&p_ready[1], 8);
    sm100::mbar_init(&o_full[0], 1);
    sm100::mbar_init(&o_full[1], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();  // (PDL) the setup above touched only shared memory, TMEM and kernel parameters
  pdl_trigger();
  const uint32_t sPa = sm100::smem_u32(sP);

  int u0 = blockIdx.x;
  if (u0 < total && unit_len(cu, heads, u0) == 0) u0 = next_unit(cu, heads, total, u0);

  if (warp == 8) {
    if (lane == 0) {
      auto issue_loads = [&](int u, int b) {
        const int bb = u / heads, h = u - bb * heads;
        const int st = cu[bb];
        uint8_t* base = bufs + b * FWD_BUF_BYTES;
        sm100::mbar_arrive_expect_tx(&load_full[b], FWD_BUF_BYTES);
        sm100::tma_load_2d(base, &tm_qkv, &load_full[b], h * d, st);
        sm100::tma_load_2d(base + TILE_BYTES, &tm_qkv, &load_full[b], H + h * d, st);
        sm100::tma_load_2d(base + 2 * TILE_BYTES, &tm_qkv, &load_full[b], 2 * H + h * d, st);
      };
      auto mma_s = [&](int i) {  // S(i): data buffer i % FWD_NBUF, TMEM S buffer i & 1
        const uint32_t q = sm100::smem_u32(bufs + (i % FWD_NBUF) * FWD_BUF_BYTES), k = q + TILE_BYTES;
        constexpr uint32_t id_s = sm100::idesc_bf16(128, 128, 0, 0);
        for (int kk = 0; kk < d / 16; ++kk)
          sm100::mma_bf16_ss(tbase + 128 * (i & 1), sm100::desc_kmajor_sw128(q + kk * 32),
                             sm100::desc_kmajor_sw128(k + kk * 32), id_s, kk > 0);
        sm100::mma_commit(&s_full[i & 1]);
      };
      auto mma_o = [&](int i) {  // O(i) = P(i) V(i): P buffer i & 1, TMEM O buffer i & 1
        const uint32_t v = sm100::smem_u32(bufs + (i % FWD_NBUF) * FWD_BUF_BYTES) + 2 * TILE_BYTES;
        const uint32_t p = sPa + (i & 1) * P_BYTES;
        constexpr uint32_t id_o = sm100::idesc_bf16(128, 64, 0, 1);
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          sm100::mma_bf16_ss(tbase + 256 + 64 * (i & 1),
                             sm100::desc_kmajor_sw128(p + (kk >> 2) * (TILE * 128) + (kk & 3) * 32),
                             sm100::desc_mnmajor_sw128(v + kk * 2048, 8192), id_o, kk > 0);
        sm100::mma_commit(&o_full[i & 1]);
      };
      // units i, i+1, i+2 of this CTA: loads run two units ahead of the MMAs
      int un[3];
      un[0] = u0;
      un[1] = un[0] < total ? next_unit(cu, heads, total, un[0]) : total;
      un[2] = un[1] < total ? next_unit(cu, heads, total, un[1]) : total;
      for (int k = 0; k < FWD_NBUF; ++k)
        if (un[k] < total) issue_loads(un[k], k);
      if (un[0] < total) {
        sm100::mbar_wait(&load_full[0], 0);
        sm100::tc_fence_after();
        mma_s(0);
      }
      for (int i = 0; un[0] < total; ++i) {
        const int nb = (i + 1) % FWD_NBUF;
        if (un[1] < total) {  // S(i+1) into the other TMEM buffer while the softmax of unit i runs
          sm100::mbar_wait(&load_full[nb], ((i + 1) / FWD_NBUF) & 1);
          sm100::tc_fence_after();
          mma_s(i + 1);
        }
        sm100::mbar_wait(&p_ready[i & 1], (i >> 1) & 1);
        sm100::tc_fence_after();
        mma_o(i);
        sm100::mbar_wait(&o_full[i & 1], (i >> 1) & 1);  // P V(i) done: data buffer i % FWD_NBUF is free
        const int u3 = un[2] < total ? next_unit(cu, heads, total, un[2]) : total;
        if (u3 < total) issue_loads(u3, i % FWD_NBUF);
        un[0] = un[1], un[1] = un[2], un[2] = u3;
      }
    }
    __syncwarp();
  } else {
    const int ch = warp >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float sc2 = rsqrtf((float)d) * LOG2E;
    // the deferred readout of unit i's O (issued as PV(i) into TMEM buffer i & 1); the O block is
    // staged in this warp's slab of P buffer i & 1, free once PV(i) has completed and until unit
    // i + 2 writes its P there (which first waits for this store to have read it)
    auto readout = [&](int i, int u, float mx, float l) {
      const uint32_t stg = sPa + (i & 1) * P_BYTES + ch * (TILE * 128) + q4 * 4096;
      const int b = u / heads, h = u - b * heads;
      const int start = cu[b];
      const int len = cu[b + 1] - start;
      sm100::mbar_wait(&o_full[i & 1], (i >> 1) & 1);
      sm100::tc_fence_after();
      float v[32];
      sm100::tmem_ld32(tbase + 256 + 64 * (i & 1) + lane_off + 32 * ch, v);
      sm100::tmem_ld_wait();
      const float inv = 1.f / l;
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] *= inv;
      if (32 * ch < d) {
        if (q4 * 32 + 32 <= len) {  // warp-uniform: all 32 rows valid -> swizzled staging + TMA store
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 pk = f32_to_bf16x8(v + 8 * c);
            st_shared_v4(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), pk.x, pk.y, pk.z, pk.w);
          }
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_2d(&tm_o, stg, h * d + 32 * ch, start + q4 * 32);
            sm100::bulk_commit();
          }
        } else if (r < len) {
          bf16* dst = O + (size_t)(start + r) * H + h * d + 32 * ch;
#pragma unroll
          for (int c = 0; c < 32; c += 8) *reinterpret_cast<uint4*>(dst + c) = f32_to_bf16x8(v + c);
        }
      }
      if (ch == 0 && r < len) lse[(size_t)h * nnz + start + r] = (mx + log2f(l)) * LN2;
      sm100::tc_fence_before();
    };
    int u_prev = -1;
    float mx_prev = 0.f, l_prev = 1.f;
    int i = 0;
    for (int u = u0; u < total; ++i) {
      const int b = u / heads, h = u - b * heads;
      const int start = cu[b];
      const int len = cu[b + 1] - start;
      const float sl2 = slopes[h] * LOG2E;
      sm100::mbar_wait(&s_full[i & 1], (i >> 1) & 1);
      sm100::tc_fence_after();
      const uint32_t tS = tbase + 128 * (i & 1) + lane_off + 64 * ch;
      float x[64];
      sm100::tmem_ld32(tS, x);
      sm100::tmem_ld32(tS + 32, x + 32);
      sm100::tmem_ld_wait();
      float mx = len == TILE ? fwd_scores<false>(x, r, ch, len, sc2, sl2) : fwd_scores<true>(x, r, ch, len, sc2, sl2);
      rmax[ch * 128 + r] = mx;
      named_bar_sync(1 + (warp & 3), 64);  // the two half-row warps only
      mx = fmaxf(rmax[r], rmax[128 + r]);
      // P = 2^(x - max) rounded to bf16 (the operand of O = P V) into P buffer i & 1 (PV(i-2), its
      // last MMA reader, finished before unit i-1's readout, whose O staging store must also have
      // read it); the row sum is taken over the rounded values
      const uint32_t pbuf = sPa + (i & 1) * P_BYTES;
      if (lane == 0) sm100::bulk_wait_read0();
      __syncwarp();
      float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int j8 = 0; j8 < 8; ++j8) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 t = __fadd2_rn(make_float2(x[j8 * 8 + 2 * e], x[j8 * 8 + 2 * e + 1]), make_float2(-mx, -mx));
          pk[e] = pack_bf16x2(ex2_approx(t.x), ex2_approx(t.y));
          sum2 = __fadd2_rn(sum2, make_float2(__uint_as_float(pk[e] << 16), __uint_as_float(pk[e] & 0xffff0000u)));
        }
        st_shared_v4(pbuf + p_off(r, 64 * ch + 8 * j8), pk[0], pk[1], pk[2], pk[3]);
      }
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&p_ready[i & 1]);
      // row sum of both halves; the two pair barriers per unit separate every rmax / rsum write
      // from the partner's previous read of it
      rsum[ch * 128 + r] = sum2.x + sum2.y;
      if (u_prev >= 0) readout(i - 1, u_prev, mx_prev, l_prev);
      named_bar_sync(1 + (warp & 3), 64);
      const float l = rsum[r] + rsum[128 + r];
      u_prev = u;
      mx_prev = mx;
      l_prev = l;
      u = next_unit(cu, heads, total, u);
    }
    if (u_prev >= 0) readout(i - 1, u_prev, mx_prev, l_prev);
    if (lane == 0) sm100::bulk_wait0();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tbase, 512);
}

// Short-sequence forward, v2 (l <= 128): the two softmax warpgroups take alternate work units
// (unit j -> warpgroup j & 1) with one thread per query row, ping-ponged on the tensor core like the
// long kernel v2: S_t = Q K^T into TMEM, P_t written back over S_t as packed bf16, O = P_t V with P
// from tensor memory, O double-buffered per warpgroup so a unit's readout runs after the next
// unit's softmax.  Q/K/V of up to four units are in flight (4 x 48 KB slots).
// A unit is one head of a GROUP of consecutive sequences whose total length fits one 128-row tile
// (several short sequences share a tile): sequences 4g..4g+3 form one group when their
// lengths sum to <= 128, else pairs 2g, 2g+1 when they fit, else single sequences.  Consecutive
// sequences are adjacent in the unpadded stream, so a group is one contiguous [<=128 x d] tile;
// each query row attends only to the key window of its own sequence (block-diagonal mask) and the
// ALiBi distance is the in-tile distance (positions restart with each sequence and both operands
// of a row-key pair are in the same sequence).
constexpr int S2_NSLOT = 4;
constexpr int S2_THREADS = SH_THREADS + 128;
constexpr int S2_UMAX = 96;  // work units per CTA (the host launches larger batches in chunks)
constexpr int S2_SMEM = S2_NSLOT * 3 * TILE_BYTES + 2 * TILE_BYTES + 1024 + 256 + 16 * S2_UMAX;  // + O staging

// Short-path work units: one head of a GROUP of consecutive sequences fitting one 128-row tile —
// sequences 4g..4g+3 when their lengths sum to <= 128, else the pair 2g, 2g+1 when it fits, else
// one sequence; empty groups are skipped.  span(b) = sequences in the group starting at b (0: none).
__device__ __forceinline__ int group_span(const int* cu, int batch, int b) {
  const int b4 = b & ~3;
  if (b4 + 3 < batch && cu[b4 + 4] - cu[b4] <= TILE) return b == b4 && cu[b4 + 4] > cu[b4] ? 4 : 0;
  const int b2 = b & ~1;
  if (b2 + 1 < batch && cu[b2 + 2] - cu[b2] <= TILE) return b == b2 && cu[b2 + 2] > cu[b2] ? 2 : 0;
  return cu[b + 1] > cu[b] ? 1 : 0;
}
// This CTA's units (candidates u = blockIdx.x + c gridDim.x, u = b * heads + h), compacted in order
// into shared memory by all NT threads: {first token, group length, h | span << 16, in-group
// sequence boundaries b1 | b2 << 8 | b3 << 16 (tile-relative, 0 when absent)}.  Walking cu per
// unit inside the roles' loops (up to six dependent reads per candidate) stalled every role.
template <int NT>
__device__ int build_group_list(const int* __restrict__ cu, int batch, int heads, int4* ulist, int* wcount) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int total = batch * heads;
  const int ncand = total > (int)blockIdx.x ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  int n = 0;
  for (int c0 = 0; c0 < ncand; c0 += NT) {
    const int c = c0 + tid;
    const int u = (int)blockIdx.x + c * (int)gridDim.x;
    int span = 0, b = 0;
    if (c < ncand) {
      b = u / heads;
      span = group_span(cu, batch, b);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, span > 0);
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int off = n;
    for (int w = 0; w < warp; ++w) off += wcount[w];
    if (span > 0) {
      const int st = cu[b];
      int bnd = 0;
      for (int e = 1; e < span; ++e) bnd |= (cu[b + e] - st) << (8 * (e - 1));
      ulist[off + __popc(bal & ((1u << lane) - 1))] = make_int4(st, cu[b + span] - st, (u - b * heads) | (span << 16), bnd);
    }
    for (int w = 0; w < NT / 32; ++w) n += wcount[w];
    __syncthreads();
  }
  return n;
}
// key window [lo, hi) of tile row r in a unit entry (its own sequence; rows past the group: [0, 1))
__device__ __forceinline__ void group_window(const int4& e, int r, int& lo, int& hi) {
  const int span = e.z >> 16;
  lo = 0;
  hi = e.y;
  for (int k = 1; k < span; ++k) {
    const int bk = (e.w >> (8 * (k - 1))) & 0xff;
    if (r >= bk) lo = bk;
    else if (hi == e.y && r < bk) hi = bk;
  }
  if (r >= e.y) lo = 0, hi = 1;
}

// ALiBi-biased scores of one query row r of a short tile, unscaled domain; keys outside the row's
// window [lo, hi) are masked when MASK; returns max_j
template <bool MASK>
__device__ __forceinline__ float row_scores_win(float (&x)[128], int r, int lo, int hi, float slr) {
  float rc = (float)r;
  asm volatile("" : "+f"(rc));  // keep the distance ramp inside the unit loop (hoisted, it spills)
  // two interleaved distance / max chains (key pairs j = 4i + 2q) instead of one 64-deep chain each
  float2 dd[2] = {make_float2(rc, rc - 1.f), make_float2(rc - 2.f, rc - 3.f)};
  float2 mx[2] = {make_float2(-INFINITY, -INFINITY), make_float2(-INFINITY, -INFINITY)};
  const uint32_t w = (uint32_t)(hi - lo);
#pragma unroll
  for (int j0 = 0; j0 < 128; j0 += 4) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = j0 + 2 * q;
      float2 t = __ffma2_rn(make_float2(fabsf(dd[q].x), fabsf(dd[q].y)), make_float2(-slr, -slr),
                            make_float2(x[j], x[j + 1]));
      dd[q] = __fadd2_rn(dd[q], make_float2(-4.f, -4.f));
      if (MASK) {
        t.x = (uint32_t)(j - lo) < w ? t.x : -INFINITY;
        t.y = (uint32_t)(j + 1 - lo) < w ? t.y : -INFINITY;
      }
      x[j] = t.x;
      x[j + 1] = t.y;
      mx[q] = make_float2(fmaxf(mx[q].x, t.x), fmaxf(mx[q].y, t.y));
    }
  }
  return fmaxf(fmaxf(mx[0].x, mx[0].y), fmaxf(mx[1].x, mx[1].y));
}

__global__ void __launch_bounds__(S2_THREADS, 1) attn_fwd_short2_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                                                                       const __grid_constant__ CUtensorMap tm_o,
                                                                       const int* __restrict__ cu, int batch, int heads,
                                                                       int d, const float* __restrict__ slopes,
                                                                       bf16* __restrict__ O, float* __restrict__ lse,
                                                                       int nnz) {
  // TMEM per warpgroup t: S_t [128 t, +128) fp32, P_t [256 + 64 t, +64) packed bf16, O_t [384 + 64 t, +64).
  // S_t is released (s_free) as soon as the warpgroup has it in registers, so S of its next unit is
  // computed during this unit's exponentials; the previous unit's O is read out after that load.
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* slots = smem;  // S2_NSLOT x (Q, K, V)
  uint8_t* sO = slots + S2_NSLOT * 3 * TILE_BYTES;  // per warpgroup t: a finished unit's O, [32 x 32] blocks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 2 * TILE_BYTES);
  uint64_t* ld_full = bars;                  // [S2_NSLOT]
  uint64_t* ld_empty = bars + S2_NSLOT;      // [S2_NSLOT]
  uint64_t* s_full = bars + 2 * S2_NSLOT;    // [2] per warpgroup
  uint64_t* s_free = s_full + 2;             // [2] per warpgroup, 4 warps arrive
  uint64_t* p_ready = s_full + 4;            // [2] per warpgroup, 4 warps arrive
  uint64_t* o_full = s_full + 6;             // [2] per warpgroup
  uint64_t* o_empty = s_full + 8;            // [2] per warpgroup, 4 warps arrive
  uint32_t* tslot = reinterpret_cast<uint32_t*>(s_full + 10);
  int4* ulist = reinterpret_cast<int4*>(s_full + 12);  // this CTA's units (build_group_list)
  __shared__ int wcount[S2_THREADS / 32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = heads * d;
  if (tid == 0) {
    sm100::tma_prefetch(&tm_qkv);
    for (int i = 0; i < S2_NSLOT; ++i) {
      sm100::mbar_init(&ld_full[i], 1);
      sm100::mbar_init(&ld_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_free[i], 4);
      sm100::mbar_init(&p_ready[i], 4);
      sm100::mbar_init(&o_full[i], 1);
      sm100::mbar_init(&o_empty[i], 4);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();
  pdl_trigger();
  const uint32_t slots_a = sm100::smem_u32(slots);
  const int nunits = build_group_list<S2_THREADS>(cu, batch, heads, ulist, wcount);

  if (warp >= 8) {
    sm100::setmaxnreg_dec<64>();
    if (warp == 9 && lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      for (int j = 0; j < nunits; ++j) {
        const int4 e = ulist[j];
        const int h = e.z & 0xffff;
#if defined(MB_DIAG_SAMELOAD)  // diagnostic builds only: every unit reads the first tile (L2-resident)
        const int st = 0;
#else
        const int st = e.x;
#endif
        const int sl = j % S2_NSLOT;
        sm100::mbar_wait(&ld_empty[sl], ((j / S2_NSLOT) & 1) ^ 1);
        uint8_t* base = slots + sl * 3 * TILE_BYTES;
        sm100::mbar_arrive_expect_tx(&ld_full[sl], 3 * TILE_BYTES);
        sm100::tma_load_2d(base, &tm_qkv, &ld_full[sl], h * d, st);
        sm100::tma_load_2d(base + TILE_BYTES, &tm_qkv, &ld_full[sl], H + h * d, st);
        sm100::tma_load_2d(base + 2 * TILE_BYTES, &tm_qkv, &ld_full[sl], 2 * H + h * d, st);
      }
    } else if (warp == 8 && lane == 0) {
      // ------------------------------------------------------------------ MMA issuer
      constexpr uint32_t id_s = sm100::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_o = sm100::idesc_bf16(128, 64, 0, 1);
      auto do_pv = [&](int i) {  // O_t = P_t V of unit i (warpgroup t = i & 1, its k-th unit)
        const int t = i & 1, k = i >> 1, sl = i % S2_NSLOT;
        sm100::mbar_wait(&o_empty[t], (k & 1) ^ 1);  // the warpgroup's previous O has been read out
        sm100::mbar_wait(&p_ready[t], k & 1);
        sm100::tc_fence_after();
        const uint32_t v = slots_a + sl * 3 * TILE_BYTES + 2 * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          sm100::mma_bf16_ts(tbase + 384 + 64 * t, tbase + 256 + 64 * t + 8 * kk,
                             sm100::desc_mnmajor_sw128(v + kk * 2048, 8192), id_o, kk > 0 ? 1u : 0u);
        sm100::mma_commit(&ld_empty[sl]);
        sm100::mma_commit(&o_full[t]);
      };
      int j = 0;
      for (; j < nunits; ++j) {
        const int t = j & 1, k = j >> 1, sl = j % S2_NSLOT;
        sm100::mbar_wait(&ld_full[sl], (j / S2_NSLOT) & 1);
        sm100::mbar_wait(&s_free[t], (k & 1) ^ 1);  // S_t of the warpgroup's previous unit is in registers
        sm100::tc_fence_after();
        const uint32_t q = slots_a + sl * 3 * TILE_BYTES, kt = q + TILE_BYTES;
        for (int kk = 0; kk < d / 16; ++kk)
          sm100::mma_bf16_ss(tbase + 128 * t, sm100::desc_kmajor_sw128(q + kk * 32),
                             sm100::desc_kmajor_sw128(kt + kk * 32), id_s, kk > 0);
        sm100::mma_commit(&s_full[t]);
        if (j >= 1) do_pv(j - 1);
      }
      if (j >= 1) do_pv(j - 1);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ softmax warpgroups
    sm100::setmaxnreg_inc<216>();
    const int t = warp >> 2, q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float sc2 = rsqrtf((float)d) * LOG2E;
    const uint32_t tS = tbase + 128 * t + lane_off, tP = tbase + 256 + 64 * t + lane_off,
                   tO = tbase + 384 + 64 * t + lane_off;
    // the previous unit's O: normalise, store, LSE; then O_t may be overwritten
    // a warp whose 32 rows are all inside the group stages its [32 x 64] block as two 64B-swizzled
    // [32 x 32] blocks in its slice of sO and one lane TMA-stores them (coalesced); a ragged quarter
    // stores its valid rows directly
    const uint32_t sOw = sm100::smem_u32(sO) + t * TILE_BYTES + q4 * 4096;
    auto readout = [&](int kk, int st, int h, int glen, float m_used, float l_used) {
      sm100::mbar_wait(&o_full[t], kk & 1);
      sm100::tc_fence_after();
      const float inv = 1.f / l_used;
      const bool full = q4 * 32 + 32 <= glen;  // warp-uniform
      bf16* dst = O + (size_t)(st + r) * H + h * d;
      if (full) {
        if (lane == 0) sm100::bulk_wait_read0();  // the previous unit's stores have left sO
        __syncwarp();
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float o[32];
        sm100::tmem_ld32(tO + 32 * hh, o);
        sm100::tmem_ld_wait();
        if (hh == 1) {
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&o_empty[t]);
        }
        if (32 * hh >= d) continue;
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] *= inv;
        if (full) {
          const uint32_t blk = sOw + hh * 2048;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 pk = f32_to_bf16x8(o + 8 * c);
            st_shared_v4(blk + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), pk.x, pk.y, pk.z, pk.w);
          }
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_2d(&tm_o, blk, h * d + 32 * hh, st + q4 * 32);
            sm100::bulk_commit();
          }
        } else if (r < glen) {
#pragma unroll
          for (int c = 0; c < 32; c += 8) *reinterpret_cast<uint4*>(dst + 32 * hh + c) = f32_to_bf16x8(o + c);
        }
      }
      if (r < glen) lse[(size_t)h * nnz + st + r] = (m_used * sc2 + __log2f(l_used)) * LN2;  // l >= 1
    };
    int j = 0, k = 0;
    int pk_k = -1, pk_st = 0, pk_h = 0, pk_glen = 0;
    float pk_m = 0.f, pk_l = 1.f;
    for (j = t; j < nunits; j += 2) {
      const int4 ue = ulist[j];
      const int st = ue.x, glen = ue.y, h = ue.z & 0xffff, span = ue.z >> 16;
      int lo, hi;
      group_window(ue, r, lo, hi);
      const float slr = slopes[h] * sqrtf((float)d);
      sm100::mbar_wait(&s_full[t], k & 1);
      sm100::tc_fence_after();
      float x[128];
#pragma unroll
      for (int i = 0; i < 4; ++i) sm100::tmem_ld32(tS + 32 * i, x + 32 * i);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&s_free[t]);  // S of the next unit may now be computed
      if (pk_k >= 0) readout(pk_k, pk_st, pk_h, pk_glen, pk_m, pk_l);  // also frees P_t (PV done)
      float m;
      if (span == 1 && glen == TILE) m = row_scores_win<false>(x, r, 0, TILE, slr);
      else m = row_scores_win<true>(x, r, lo, hi, slr);
      const float nm = -m * sc2;
      float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // two row-sum chains
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float pk[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int c = 64 * hh + 2 * q;
          const float2 tt = __ffma2_rn(make_float2(x[c], x[c + 1]), make_float2(sc2, sc2), make_float2(nm, nm));
          const float2 e = make_float2(ex2_approx(tt.x), ex2_approx(tt.y));
          ls[q & 1] = __fadd2_rn(ls[q & 1], e);
          pk[q] = __uint_as_float(pack_bf16x2(e.x, e.y));
        }
        sm100::tmem_st32(tP + 32 * hh, pk);
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&p_ready[t]);
      pk_k = k, pk_st = st, pk_h = h, pk_glen = glen, pk_m = m, pk_l = (ls[0].x + ls[1].x) + (ls[0].y + ls[1].y);
      ++k;
    }
    if (pk_k >= 0) readout(pk_k, pk_st, pk_h, pk_glen, pk_m, pk_l);
    if (lane == 0) sm100::bulk_wait0();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tbase, 512);
}

// Long-forward scores in the unscaled domain y = S - (m_h / sc) |q - k| (sc = log2e / sqrt(d) is
// applied inside the exponent, P = 2^(sc y - sc max y)); distances stepped by -2 per key pair so
// no per-pair constants are materialised.  Returns max_j y (-inf past the sequence when MASK).
template <bool MASK>
__device__ __forceinline__ float lf_scores(float (&x)[64], int r, int ch, int keys, float slr, int qk_off) {
  const float rc = (float)(r + qk_off - 64 * ch);
  float2 dd = make_float2(rc, rc - 1.f);
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 64; j += 2) {
    const float2 t = __ffma2_rn(make_float2(fabsf(dd.x), fabsf(dd.y)), make_float2(-slr, -slr),
                                make_float2(x[j], x[j + 1]));
    dd = __fadd2_rn(dd, make_float2(-2.f, -2.f));
    x[j] = t.x;
    x[j + 1] = t.y;
    if (MASK) {
      x[j] = 64 * ch + j < keys ? x[j] : -INFINITY;
      x[j + 1] = 64 * ch + j + 1 < keys ? x[j + 1] : -INFINITY;
    }
    mx = fmaxf(mx, fmaxf(x[j], x[j + 1]));
  }
  return mx;
}

// Long-sequence forward (128 < l <= 2048, SURVEY A5 at l = 512 and F4): one work unit = (128-row
// query tile, head, sequence), iterating over the sequence's key tiles with the online softmax,
// starting at the diagonal tile (where ALiBi puts the row maxima).  Warp 9 (one lane) streams Q
// (double-buffered per unit) and K/V tiles (LF_NS-stage ring) by TMA; warp 8 (one lane) issues
// S_{g+1} = Q K_{g+1}^T into the other half of a double-buffered TMEM S while the softmax warps work
// on S_g, then O += P_g V_g and l += P_g 1 (an N=16 MMA against an all-ones tile) straight into the
// unit's TMEM accumulators (double-buffered per unit).  Warps 0-7 (two threads per query row, 64
// keys each) keep the running max the P tiles were computed against and rescale the TMEM
// accumulators only when a row's max grows by more than 2^8 (rare once the diagonal tile has set
// it); a unit's O is normalised and stored during the next unit's first tile, so no MMA latency is
// exposed at unit boundaries.  TMEM: S [0,256) (2 x 128), O [256,384) (2 x 64), l [384,416) (2 x 16).
// ------------------------------------------------------------------------------------------
constexpr int LF_NS = 3;
constexpr int LF_THREADS = SH_THREADS + 64;
constexpr int ONES_BYTES = 16 * TILE * 2;  // [16 x 128] bf16 ones: B operand of the row-sum MMA
constexpr int LF_SMEM = 2 * TILE_BYTES + LF_NS * 2 * TILE_BYTES + 2 * P_BYTES + ONES_BYTES + 1024 + 256;

struct LongUnits {  // unit u = (b * heads + h) * QT + qt, valid iff qt * 128 < len_b
  const int* cu;
  int heads, QT, total;
  __device__ __forceinline__ bool valid(int u) const {
    const int b = u / (heads * QT), qt = u % QT;
    return qt * TILE < cu[b + 1] - cu[b];
  }
  __device__ __forceinline__ int next(int u) const {
    for (u += gridDim.x; u < total; u += gridDim.x)
      if (valid(u)) return u;
    return total;
  }
  __device__ __forceinline__ int first() const {
    int u = blockIdx.x;
    if (u < total && !valid(u)) u = next(u);
    return u;
  }
  __device__ __forceinline__ void decode(int u, int& b, int& h, int& qt) const {
    b = u / (heads * QT);
    const int rem = u - b * heads * QT;
    h = rem / QT;
    qt = rem - h * QT;
  }
};

__global__ void __launch_bounds__(LF_THREADS, 1) attn_fwd_long_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                                                                     const __grid_constant__ CUtensorMap tm_o,
                                                                     LongUnits U, int d,
                                                                     const float* __restrict__ slopes,
                                                                     bf16* __restrict__ O, float* __restrict__ lse,
                                                                     int nnz) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                              // 2 x Q
  uint8_t* sKV = sQ + 2 * TILE_BYTES;              // LF_NS x (K, V)
  uint8_t* sP = sKV + LF_NS * 2 * TILE_BYTES;
  uint8_t* sOnes = sP + 2 * P_BYTES;  // sP: two P buffers (tile g uses g & 1)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOnes + ONES_BYTES);
  uint64_t* q_full = bars;                         // [2]
  uint64_t* q_empty = bars + 2;                    // [2]
  uint64_t* kv_full = bars + 4;                    // [LF_NS]
  uint64_t* kv_empty = bars + 4 + LF_NS;           // [LF_NS]
  uint64_t* s_full = bars + 4 + 2 * LF_NS;         // [2]
  uint64_t* pv_full = bars + 6 + 2 * LF_NS;        // [2] per tile: PV_g (and l_g) accumulated
  uint64_t* p_ready = bars + 8 + 2 * LF_NS;        // [2] by tile parity, 8 softmax warps (see the short kernel)
  uint64_t* o_done = bars + 10 + 2 * LF_NS;        // [2] per unit: its last PV accumulated
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 12 + 2 * LF_NS);
  __shared__ float rmax[2][2 * TILE];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = U.heads * d;
  if (tid == 0) {
    sm100::tma_prefetch(&tm_qkv);
    sm100::tma_prefetch(&tm_o);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&q_full[i], 1);
      sm100::mbar_init(&q_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&pv_full[i], 1);
      sm100::mbar_init(&o_done[i], 1);
    }
    for (int i = 0; i < LF_NS; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
    }
    sm100::mbar_init(&p_ready[0], 8);
    sm100::mbar_init(&p_ready[1], 8);
    sm100::fence_barrier_init();
  }
  for (int i = tid; i < ONES_BYTES / 16; i += LF_THREADS)  // bf16 1.0 = 0x3F80 (any swizzle of ones is ones)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  sm100::fence_proxy_async_smem();
  if (warp == 0) sm100::tmem_alloc(tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();  // (PDL) the setup above touched only shared memory, TMEM and kernel parameters
  pdl_trigger();
  const uint32_t sQa = sm100::smem_u32(sQ), sKVa = sm100::smem_u32(sKV), sPa = sm100::smem_u32(sP),
                 sOa = sm100::smem_u32(sOnes);
  auto nkv_of = [&](int u) {
    int b, h, qt;
    U.decode(u, b, h, qt);
    return (U.cu[b + 1] - U.cu[b] + TILE - 1) / TILE;
  };

  if (warp == 9) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int uc = 0, g = 0;
      for (int u = U.first(); u < U.total; u = U.next(u), ++uc) {
        int b, h, qt;
        U.decode(u, b, h, qt);
        const int st = U.cu[b], nkv = (U.cu[b + 1] - st + TILE - 1) / TILE;
        const int qb = uc & 1;
        sm100::mbar_wait(&q_empty[qb], ((uc >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&q_full[qb], TILE_BYTES);
        sm100::tma_load_2d(sQ + qb * TILE_BYTES, &tm_qkv, &q_full[qb], h * d, st + qt * TILE);
        for (int jj = 0; jj < nkv; ++jj, ++g) {
          const int j = (qt + jj) % nkv;  // diagonal tile first
          const int sg = g % LF_NS;
          sm100::mbar_wait(&kv_empty[sg], ((g / LF_NS) & 1) ^ 1);
          uint8_t* kv = sKV + sg * 2 * TILE_BYTES;
          sm100::mbar_arrive_expect_tx(&kv_full[sg], 2 * TILE_BYTES);
          sm100::tma_load_2d(kv, &tm_qkv, &kv_full[sg], H + h * d, st + j * TILE);
          sm100::tma_load_2d(kv + TILE_BYTES, &tm_qkv, &kv_full[sg], 2 * H + h * d, st + j * TILE);
        }
      }
    }
    __syncwarp();
  } else if (warp == 8) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_s = sm100::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_o = sm100::idesc_bf16(128, 64, 0, 1);
      constexpr uint32_t id_l = sm100::idesc_bf16(128, 16, 0, 0);
      // (unit, tile) cursor over this CTA's flattened tile sequence
      int u = U.first(), uc = 0, j = 0, nkv = u < U.total ? nkv_of(u) : 0;
      auto issue_s = [&](int g, int uu_c, int last) {  // S_g = Q K_g^T into S buffer g & 1
        const int sg = g % LF_NS;
        sm100::mbar_wait(&kv_full[sg], (g / LF_NS) & 1);
        sm100::tc_fence_after();
        const uint32_t q = sQa + (uu_c & 1) * TILE_BYTES, k = sKVa + sg * 2 * TILE_BYTES;
        for (int kk = 0; kk < d / 16; ++kk)
          sm100::mma_bf16_ss(tbase + 128 * (g & 1), sm100::desc_kmajor_sw128(q + kk * 32),
                             sm100::desc_kmajor_sw128(k + kk * 32), id_s, kk > 0);
        sm100::mma_commit(&s_full[g & 1]);
        if (last) sm100::mma_commit(&q_empty[uu_c & 1]);  // the unit's last read of its Q
      };
      if (u < U.total) {
        sm100::mbar_wait(&q_full[0], 0);
        issue_s(0, 0, nkv == 1);
      }
      for (int g = 0; u < U.total; ++g) {
        // cursor of tile g + 1
        int u2 = u, uc2 = uc, j2 = j + 1, nkv2 = nkv;
        if (j2 == nkv) {
          u2 = U.next(u);
          ++uc2;
          j2 = 0;
          nkv2 = u2 < U.total ? nkv_of(u2) : 0;
        }
        if (u2 < U.total) {
          if (j2 == 0) sm100::mbar_wait(&q_full[uc2 & 1], (uc2 >> 1) & 1);
          issue_s(g + 1, uc2, j2 == nkv2 - 1);
        }
        sm100::mbar_wait(&p_ready[g & 1], (g >> 1) & 1);  // P_g in smem (S_g consumed)
        sm100::tc_fence_after();
        const uint32_t v = sKVa + (g % LF_NS) * 2 * TILE_BYTES + TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk) {  // O += P V, l += P 1 into the unit's accumulators
          const uint64_t pa = sm100::desc_kmajor_sw128(sPa + (g & 1) * P_BYTES + (kk >> 2) * (TILE * 128) + (kk & 3) * 32);
          const uint32_t acc = (j > 0 || kk > 0) ? 1u : 0u;
          sm100::mma_bf16_ss(tbase + 256 + 64 * (uc & 1), pa, sm100::desc_mnmajor_sw128(v + kk * 2048, 8192), id_o,
                             acc);
          sm100::mma_bf16_ss(tbase + 384 + 16 * (uc & 1), pa,
                             sm100::desc_kmajor_sw128(sOa + (kk >> 2) * 2048 + (kk & 3) * 32), id_l, acc);
        }
        sm100::mma_commit(&pv_full[g & 1]);
        sm100::mma_commit(&kv_empty[g % LF_NS]);
        if (j + 1 == nkv) sm100::mma_commit(&o_done[uc & 1]);
        u = u2, uc = uc2, j = j2, nkv = nkv2;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ softmax warps 0-7
    const int ch = warp >> 2, q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float sc2 = rsqrtf((float)d) * LOG2E;
    const float tau = 8.f / sc2;  // rescale only when a row max grows by more than 2^8 in P
    // the deferred epilogue of a finished unit: O / l from its TMEM accumulators, stored as bf16 O
    // (staged in the retired P buffer `pb`) and the LSE
    auto epilogue = [&](int uu, int ucc, float m_used, uint32_t pb) {
      int b, h, qt;
      U.decode(uu, b, h, qt);
      const int start = U.cu[b], len = U.cu[b + 1] - start, q0 = qt * TILE;
      sm100::mbar_wait(&o_done[ucc & 1], (ucc >> 1) & 1);
      sm100::tc_fence_after();
      float o[32];
      sm100::tmem_ld32(tbase + 256 + 64 * (ucc & 1) + lane_off + 32 * ch, o);
      const float lt = sm100::tmem_ld1(tbase + 384 + 16 * (ucc & 1) + lane_off);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      const float inv = 1.f / lt;
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] *= inv;
      const int qrow = q0 + r;
      if (32 * ch < d) {
        if (q0 + q4 * 32 + 32 <= len) {  // warp-uniform: all 32 rows valid -> swizzled staging + TMA store
          const uint32_t stg = pb + ch * (TILE * 128) + q4 * 4096;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 pk = f32_to_bf16x8(o + 8 * c);
            st_shared_v4(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), pk.x, pk.y, pk.z, pk.w);
          }
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_2d(&tm_o, stg, h * d + 32 * ch, start + q0 + q4 * 32);
            sm100::bulk_commit();
          }
        } else if (qrow < len) {
          bf16* dst = O + (size_t)(start + qrow) * H + h * d + 32 * ch;
#pragma unroll
          for (int c = 0; c < 32; c += 8) *reinterpret_cast<uint4*>(dst + c) = f32_to_bf16x8(o + c);
        }
      }
      if (ch == 0 && qrow < len) lse[(size_t)h * nnz + start + qrow] = (m_used * sc2 + log2f(lt)) * LN2;
    };
    int g = 0, uc = 0;
    int pend_u = -1, pend_uc = 0;  // unit whose epilogue is pending
    float pend_m = 0.f;
    for (int u = U.first(); u < U.total; u = U.next(u), ++uc) {
      int b, h, qt;
      U.decode(u, b, h, qt);
      const int start = U.cu[b], len = U.cu[b + 1] - start, q0 = qt * TILE;
      (void)start;
      const int nkv = (len + TILE - 1) / TILE;
      const float slr = slopes[h] * sqrtf((float)d);  // m_h / (1/sqrt(d)): bias in the unscaled domain
      float m = -INFINITY;  // the max the unit's P tiles are computed against (unscaled domain)
      for (int jj = 0; jj < nkv; ++jj, ++g) {
        const int kv0 = ((qt + jj) % nkv) * TILE;
        sm100::mbar_wait(&s_full[g & 1], (g >> 1) & 1);
        sm100::tc_fence_after();
        float x[64];
        const uint32_t tS = tbase + 128 * (g & 1) + lane_off + 64 * ch;
        sm100::tmem_ld32(tS, x);
        sm100::tmem_ld32(tS + 32, x + 32);
        sm100::tmem_ld_wait();
        const float mx = len - kv0 >= TILE ? lf_scores<false>(x, r, ch, len - kv0, slr, q0 - kv0)
                                           : lf_scores<true>(x, r, ch, len - kv0, slr, q0 - kv0);
        rmax[g & 1][ch * TILE + r] = mx;
        named_bar_sync(1 + (warp & 3), 64);  // the two half-row warps only
        const float m_row = fmaxf(rmax[g & 1][r], rmax[g & 1][TILE + r]);
        if (jj == 0) {
          m = m_row;
        } else if (__any_sync(0xffffffffu, m_row > m + tau)) {
          // some row of this warp outgrew its max: rescale its O / l accumulators (after PV_{g-1})
          const float m_new = fmaxf(m, m_row);
          const float alpha = ex2_approx((m - m_new) * sc2);
          sm100::mbar_wait(&pv_full[(g - 1) & 1], ((g - 1) >> 1) & 1);
          sm100::tc_fence_after();
          float o[32];
          const uint32_t to = tbase + 256 + 64 * (uc & 1) + lane_off + 32 * ch;
          sm100::tmem_ld32(to, o);
          float lv[1];
          lv[0] = sm100::tmem_ld1(tbase + 384 + 16 * (uc & 1) + lane_off);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= alpha;
          sm100::tmem_st32(to, o);
          if (ch == 0) sm100::tmem_st1(tbase + 384 + 16 * (uc & 1) + lane_off, lv[0] * alpha);  // warp-uniform
          sm100::tmem_st_wait();
          m = m_new;
        }
        // P_g = 2^(sc (y - m)) rounded to bf16 into P buffer g & 1 (PV_{g-2}, its last reader, done;
        // any O staging store from it has been read)
        if (g >= 2) sm100::mbar_wait(&pv_full[g & 1], ((g - 2) >> 1) & 1);
        if (lane == 0) sm100::bulk_wait_read0();
        __syncwarp();
        const float nm = -m * sc2;
        const uint32_t pbuf = sPa + (g & 1) * P_BYTES;
#pragma unroll
        for (int j8 = 0; j8 < 8; ++j8) {
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 t = __ffma2_rn(make_float2(x[j8 * 8 + 2 * e], x[j8 * 8 + 2 * e + 1]), make_float2(sc2, sc2),
                                        make_float2(nm, nm));
            pk[e] = pack_bf16x2(ex2_approx(t.x), ex2_approx(t.y));
          }
          st_shared_v4(pbuf + p_off(r, 64 * ch + 8 * j8), pk[0], pk[1], pk[2], pk[3]);
        }
        sm100::fence_proxy_async_smem();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&p_ready[g & 1]);
        if (jj == 0 && pend_u >= 0) {  // the previous unit's epilogue, its O staged in its last P buffer
          epilogue(pend_u, pend_uc, pend_m, sPa + ((g - 1) & 1) * P_BYTES);
          pend_u = -1;
        }
      }
      pend_u = u;
      pend_uc = uc;
      pend_m = m;
    }
    if (pend_u >= 0) epilogue(pend_u, pend_uc, pend_m, sPa + ((g - 1) & 1) * P_BYTES);
    if (lane == 0) sm100::bulk_wait0();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tbase, 512);
}

// Long-sequence forward, v2: two query tiles per unit, ping-ponged (the FlashAttention-4 schedule
// on sm_100a).  A unit = (query tiles 2p and 2p+1, head, sequence); the two tiles share every K/V
// tile the TMA warp streams in.  Softmax warpgroup t (warps 4t..4t+3) owns query tile t with ONE
// thread per query row (128 keys per thread: no cross-thread row-max exchange).  The MMA warp issues
// S_t = Q_t K^T into TMEM; warpgroup t loads S_t into registers and releases it at once (so S_t of
// the next key tile is computed while this tile's exponentials run), adds the ALiBi bias,
// exponentiates in the exp2 domain and writes P_t as packed bf16 into its own TMEM columns; O_t +=
// P_t V then runs with A = P_t straight from tensor memory (tcgen05.mma A-in-TMEM), so P never
// touches shared memory.  The row sum l stays in registers (fp32); the O accumulators are rescaled
// only when a row max grows by more than 2^8 (rare with the diagonal key tile first).  A unit's O is
// normalised and stored right after the first key tile of the next unit has been loaded.  Each CTA
// builds its unit list once in shared memory.
// TMEM: S_t [128 t, +128), P_t [256 + 64 t, +64) (bf16 pairs), O_t [384 + 64 t, +64).
constexpr int L2_NS = 3;
constexpr int L2_THREADS = SH_THREADS + 128;  // softmax warpgroups 0, 1; warpgroup 2: MMA warp 8, TMA warp 9
constexpr int L2_UMAX = 2048;                 // work units per CTA (host falls back to v1 beyond)
constexpr int L2_SMEM = 4 * TILE_BYTES + L2_NS * 2 * TILE_BYTES + 2 * TILE_BYTES + 1024 + 256 + 16 * L2_UMAX;  // + O staging

struct PairUnits {  // unit u = (b * heads + h) * QP + p, valid iff 256 p < len_b
  const int* cu;
  int heads, QP, total;
};

// ALiBi-biased scores of one full query row (128 keys, one thread per row), unscaled domain:
// x_j += -slr |(r + qk_off) - j|, keys at or past `keys` masked when MASK; returns max_j.
// Two interleaved distance / max chains (key pairs j = 4i + 2q, q = 0, 1) so that neither the
// distance update nor the running max is a 64-deep dependency chain.
template <bool MASK>
__device__ __forceinline__ float row_scores128(float (&x)[128], int r, int keys, float slr, int qk_off) {
  const float rc = (float)(r + qk_off);
  float2 dd[2], mx[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    dd[q] = make_float2(rc - (float)(2 * q), rc - (float)(2 * q + 1));
    mx[q] = make_float2(-INFINITY, -INFINITY);
  }
#pragma unroll
  for (int j0 = 0; j0 < 128; j0 += 4) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = j0 + 2 * q;
      float2 t = __ffma2_rn(make_float2(fabsf(dd[q].x), fabsf(dd[q].y)), make_float2(-slr, -slr),
                            make_float2(x[j], x[j + 1]));
      dd[q] = __fadd2_rn(dd[q], make_float2(-4.f, -4.f));
      if (MASK) {
        t.x = j < keys ? t.x : -INFINITY;
        t.y = j + 1 < keys ? t.y : -INFINITY;
      }
      x[j] = t.x;
      x[j + 1] = t.y;
      mx[q] = make_float2(fmaxf(mx[q].x, t.x), fmaxf(mx[q].y, t.y));
    }
  }
  return fmaxf(fmaxf(mx[0].x, mx[0].y), fmaxf(mx[1].x, mx[1].y));
}

#ifdef MB_TRACE_L2
// diagnostic builds only: clock64 stamps of CTA 0's phases over key tiles [TR0, TR0 + 16)
constexpr int TR0 = 40;
__device__ long long l2_trace[2][16][8];  // per warpgroup: wait S, S in, S loaded, scores, pv waited, exps, p_ready
__device__ long long l2_mtrace[2][8][16];  // per t: S_t issued, PV_t issued, S: enter, kv ok; PV: enter
#define L2TR(t_, c_, ev_)                                                                  \
  do {                                                                                     \
    if (blockIdx.x == 0 && (c_) >= TR0 && (c_) < TR0 + 16) l2_trace[t_][(c_) - TR0][ev_] = clock64(); \
  } while (0)
#define L2MTR(t_, k_, c_)                                                                  \
  do {                                                                                     \
    if (blockIdx.x == 0 && (c_) >= TR0 && (c_) < TR0 + 16) l2_mtrace[t_][k_][(c_) - TR0] = clock64(); \
  } while (0)
#else
#define L2TR(t_, c_, ev_) \
  do {                    \
  } while (0)
#define L2MTR(t_, k_, c_) \
  do {                    \
  } while (0)
#endif

__global__ void __launch_bounds__(L2_THREADS, 1) attn_fwd_long2_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                                                                      const __grid_constant__ CUtensorMap tm_o,
                                                                      PairUnits U, int d,
                                                                      const float* __restrict__ slopes,
                                                                      bf16* __restrict__ O, float* __restrict__ lse,
                                                                      int nnz) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // [unit parity][tile] Q
  uint8_t* sKV = sQ + 4 * TILE_BYTES;  // L2_NS x (K, V)
  uint8_t* sO = sKV + L2_NS * 2 * TILE_BYTES;  // per warpgroup t: the finished unit's O, [32 x 32] blocks
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + 2 * TILE_BYTES);
  uint64_t* q_full = bars;                  // [2] per unit parity
  uint64_t* q_empty = bars + 2;             // [2]
  uint64_t* kv_full = bars + 4;             // [L2_NS]
  uint64_t* kv_empty = bars + 4 + L2_NS;    // [L2_NS]
  uint64_t* s_full = bars + 4 + 2 * L2_NS;  // [2] per query tile t
  uint64_t* s_free = s_full + 2;            // [2] per t, 4 warps arrive: S_t is in registers
  uint64_t* p_ready = s_full + 4;           // [2] per t, 4 warps arrive
  uint64_t* pv_done = s_full + 6;           // [2] per t, one phase per PV_t
  uint32_t* tslot = reinterpret_cast<uint32_t*>(s_full + 8);
  int4* ulist = reinterpret_cast<int4*>(s_full + 10);  // {st, len, h | p << 16, two}
  __shared__ int wcount[L2_THREADS / 32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = U.heads * d;
  if (tid == 0) {
    sm100::tma_prefetch(&tm_qkv);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&q_full[i], 1);
      sm100::mbar_init(&q_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_free[i], 4);
      sm100::mbar_init(&p_ready[i], 4);
      sm100::mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < L2_NS; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();
  pdl_trigger();
  const uint32_t sQa = sm100::smem_u32(sQ), sKVa = sm100::smem_u32(sKV);
  // this CTA's unit list (candidates blockIdx.x + c gridDim.x), compacted once by all threads
  const int ncand = U.total > (int)blockIdx.x ? (U.total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  int nunits = 0;
  for (int c0 = 0; c0 < ncand; c0 += L2_THREADS) {
    const int c = c0 + tid;
    const int u = (int)blockIdx.x + c * (int)gridDim.x;
    int st = 0, len = 0, h = 0, p = 0;
    bool ok = false;
    if (c < ncand) {
      const int b = u / (U.heads * U.QP);
      const int rem = u - b * U.heads * U.QP;
      h = rem / U.QP;
      p = rem - h * U.QP;
      st = U.cu[b];
      len = U.cu[b + 1] - st;
      ok = p * 2 * TILE < len;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int off = nunits;
    for (int w = 0; w < warp; ++w) off += wcount[w];
    if (ok) ulist[off + __popc(bal & ((1u << lane) - 1))] = make_int4(st, len, h | (p << 16), (2 * p + 1) * TILE < len);
    for (int w = 0; w < L2_THREADS / 32; ++w) nunits += wcount[w];
    __syncthreads();
  }

  // registers: 12 warps leave 168 per thread; the producer/issuer warpgroup (warps 8-11) hands most
  // of its share to the two softmax warpgroups (a full 128-key score row per thread lives in registers)
  if (warp >= 8) {
    sm100::setmaxnreg_dec<64>();
    if (warp == 9 && lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      int g = 0;
      for (int uc = 0; uc < nunits; ++uc) {
        const int4 e = ulist[uc];
        const int st = e.x, len = e.y, h = e.z & 0xffff, p = e.z >> 16;
        const bool two = e.w;
        const int nkv = (len + TILE - 1) / TILE;
        const int qb = uc & 1;
        sm100::mbar_wait(&q_empty[qb], ((uc >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&q_full[qb], (two ? 2 : 1) * TILE_BYTES);
        sm100::tma_load_2d(sQ + 2 * qb * TILE_BYTES, &tm_qkv, &q_full[qb], h * d, st + 2 * p * TILE);
        if (two) sm100::tma_load_2d(sQ + (2 * qb + 1) * TILE_BYTES, &tm_qkv, &q_full[qb], h * d, st + (2 * p + 1) * TILE);
        for (int jj = 0; jj < nkv; ++jj, ++g) {
          const int j = (2 * p + jj) % nkv;  // query tile 0's diagonal key tile first
          const int sg = g % L2_NS;
          sm100::mbar_wait(&kv_empty[sg], ((g / L2_NS) & 1) ^ 1);
          uint8_t* kv = sKV + sg * 2 * TILE_BYTES;
          sm100::mbar_arrive_expect_tx(&kv_full[sg], 2 * TILE_BYTES);
          sm100::tma_load_2d(kv, &tm_qkv, &kv_full[sg], H + h * d, st + j * TILE);
          sm100::tma_load_2d(kv + TILE_BYTES, &tm_qkv, &kv_full[sg], 2 * H + h * d, st + j * TILE);
        }
      }
    } else if (warp == 8) {  // the whole warp runs the issue loop; one elected lane issues
      // ------------------------------------------------------------------ MMA issuer
      constexpr uint32_t id_s = sm100::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_o = sm100::idesc_bf16(128, 64, 0, 1);
      int c[2] = {0, 0}, sc[2] = {0, 0};  // PVs / S issued per query tile t
      auto issue_s = [&](int t, uint32_t q, int sg) {  // S_t = Q_t K_sg^T, once S_t's last tile is in registers
        L2MTR(t, 3, sc[t]);
        sm100::mbar_wait(&s_free[t], (sc[t] & 1) ^ 1);
        L2MTR(t, 0, sc[t]);
        ++sc[t];
        sm100::tc_fence_after();
        const uint32_t k = sKVa + sg * 2 * TILE_BYTES;
        for (int kk = 0; kk < d / 16; ++kk)
          sm100::mma_bf16_ss_w(tbase + 128 * t, sm100::desc_kmajor_sw128(q + kk * 32), sm100::desc_kmajor_sw128(k + kk * 32),
                             id_s, kk > 0);
        L2MTR(t, 5, sc[t] - 1);
        sm100::mma_commit_w(&s_full[t]);
      };
      auto issue_pv = [&](int t, int sg, bool acc) {  // O_t += P_t V_sg (P_t from TMEM), after P_t is written
        L2MTR(t, 4, c[t]);
        sm100::mbar_wait(&p_ready[t], c[t] & 1);
        L2MTR(t, 1, c[t]);
        sm100::tc_fence_after();
        const uint32_t v = sKVa + sg * 2 * TILE_BYTES + TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          sm100::mma_bf16_ts_w(tbase + 384 + 64 * t, tbase + 256 + 64 * t + 8 * kk,
                             sm100::desc_mnmajor_sw128(v + kk * 2048, 8192), id_o, (acc || kk > 0) ? 1u : 0u);
        L2MTR(t, 6, c[t]);
        sm100::mma_commit_w(&pv_done[t]);
        ++c[t];
      };
      // flattened key-tile sequence over this CTA's units: S_t of tile g + 1 is issued as soon as
      // warpgroup t holds S_t(g) in registers (before PV_t(g)), so it overlaps the exponentials
      auto unit_two = [&](int uc) { return ulist[uc].w != 0; };
      auto unit_nkv = [&](int uc) { return (ulist[uc].y + TILE - 1) / TILE; };
      auto issue_s_tile = [&](int t, int uc, int g) {  // S_t of global tile g (unit uc)
        const int sg = g % L2_NS;
        L2MTR(t, 2, sc[t]);
        if (t == 0) {
          sm100::mbar_wait(&kv_full[sg], (g / L2_NS) & 1);
          sm100::tc_fence_after();
        }
        issue_s(t, sQa + (2 * (uc & 1) + t) * TILE_BYTES, sg);
      };
      if (nunits > 0) {
        sm100::mbar_wait(&q_full[0], 0);
        issue_s_tile(0, 0, 0);
        if (unit_two(0)) issue_s_tile(1, 0, 0);
      }
      int g = 0;
      for (int uc = 0; uc < nunits; ++uc) {
        const bool two = unit_two(uc);
        const int nkv = unit_nkv(uc);
        for (int jj = 0; jj < nkv; ++jj, ++g) {
          // the next tile of the flattened sequence
          int nu = uc, nj = jj + 1;
          if (nj == nkv) {
            nu = uc + 1;
            nj = 0;
          }
          const bool has_next = nu < nunits;
          const bool next_two = has_next && unit_two(nu);
          if (has_next) {
            if (nj == 0) sm100::mbar_wait(&q_full[nu & 1], (nu >> 1) & 1);
            issue_s_tile(0, nu, g + 1);
          }
          issue_pv(0, g % L2_NS, jj > 0);
          if (next_two) issue_s_tile(1, nu, g + 1);
          if (two) issue_pv(1, g % L2_NS, jj > 0);
          sm100::mma_commit_w(&kv_empty[g % L2_NS]);
        }
        sm100::mma_commit_w(&q_empty[uc & 1]);  // every S of this unit has been issued
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ softmax warpgroups
    sm100::setmaxnreg_inc<216>();  // 2 x 128 x 216 + 128 x 64 <= 384 x 168
    const int t = warp >> 2, q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float sc2 = rsqrtf((float)d) * LOG2E;
    const float tau = 8.f / sc2;  // rescale only when a row max grows by more than 2^8 in P
    const uint32_t tS = tbase + 128 * t + lane_off, tP = tbase + 256 + 64 * t + lane_off,
                   tO = tbase + 384 + 64 * t + lane_off;
    int c = 0;  // key tiles processed by this warpgroup (all units)
    // a finished unit's O: normalise, store, LSE (its last PV is pv_done phase c - 1)
    // a warp whose 32 rows are all inside the sequence stages its [32 x 64] block as two 64B-swizzled
    // [32 x 32] blocks in its slice of sO and one lane TMA-stores them (coalesced); a ragged quarter
    // stores its valid rows directly
    const uint32_t sOw = sm100::smem_u32(sO) + t * TILE_BYTES + q4 * 4096;
    auto readout = [&](int st, int len, int h, int qrow, float m_used, float l_used) {
      sm100::mbar_wait(&pv_done[t], (c - 1) & 1);
      sm100::tc_fence_after();
      const float inv = 1.f / l_used;
      const int qbase = qrow - lane;                  // first row of this warp's quarter
      const bool full = qbase + 32 <= len;           // warp-uniform
      bf16* dst = O + (size_t)(st + qrow) * H + h * d;
      if (full) {
        if (lane == 0) sm100::bulk_wait_read0();     // the previous unit's stores have left sO
        __syncwarp();
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float o[32];
        sm100::tmem_ld32(tO + 32 * hh, o);
        sm100::tmem_ld_wait();
        if (32 * hh >= d) continue;
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] *= inv;
        if (full) {
          const uint32_t blk = sOw + hh * 2048;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const uint4 pk = f32_to_bf16x8(o + 8 * cc);
            st_shared_v4(blk + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4), pk.x, pk.y, pk.z, pk.w);
          }
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_2d(&tm_o, blk, h * d + 32 * hh, st + qbase);
            sm100::bulk_commit();
          }
        } else if (qrow < len) {
#pragma unroll
          for (int cc = 0; cc < 32; cc += 8) *reinterpret_cast<uint4*>(dst + 32 * hh + cc) = f32_to_bf16x8(o + cc);
        }
      }
      if (qrow < len) lse[(size_t)h * nnz + st + qrow] = (m_used * sc2 + __log2f(l_used)) * LN2;  // l >= 1
    };
    bool pend = false;
    int pd_st = 0, pd_len = 0, pd_h = 0, pd_row = 0;
    float pd_m = 0.f, pd_l = 1.f;
    for (int uc = 0; uc < nunits; ++uc) {
      const int4 e = ulist[uc];
      const int st = e.x, len = e.y, h = e.z & 0xffff, p = e.z >> 16;
      if (t == 1 && !e.w) continue;  // no second query tile in this unit
      const int nkv = (len + TILE - 1) / TILE;
      const int q0 = (2 * p + t) * TILE;
      const float slr = slopes[h] * sqrtf((float)d);  // m_h / (1/sqrt(d)): bias in the unscaled domain
      float m = -INFINITY, l = 0.f;
      for (int jj = 0; jj < nkv; ++jj) {
        const int kv0 = ((2 * p + jj) % nkv) * TILE;
        const bool trw = q4 == 0 && lane == 0;
        if (trw) L2TR(t, c, 0);
        sm100::mbar_wait(&s_full[t], c & 1);
        if (trw) L2TR(t, c, 1);
        sm100::tc_fence_after();
        float x[128];
#pragma unroll
        for (int i = 0; i < 4; ++i) sm100::tmem_ld32(tS + 32 * i, x + 32 * i);
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&s_free[t]);
        if (trw) L2TR(t, c, 2);
        const int keys = len - kv0;
        const float mx = keys >= TILE ? row_scores128<false>(x, r, keys, slr, q0 - kv0)
                                      : row_scores128<true>(x, r, keys, slr, q0 - kv0);
        if (jj == 0 && pend) {  // the previous unit's O: after this tile's score pass its last PV is done
          readout(pd_st, pd_len, pd_h, pd_row, pd_m, pd_l);
          pend = false;
        }
        if (trw) L2TR(t, c, 3);
        if (jj > 0) {
          // P_t of the previous key tile must have been consumed before P_t is rewritten, and a
          // rescale of O_t must follow that PV
          sm100::mbar_wait(&pv_done[t], (c - 1) & 1);
          if (__any_sync(0xffffffffu, mx > m + tau)) {
            const float m_new = fmaxf(m, mx);
            const float alpha = ex2_approx((m - m_new) * sc2);
            sm100::tc_fence_after();
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float o[32];
              sm100::tmem_ld32(tO + 32 * hh, o);
              sm100::tmem_ld_wait();
#pragma unroll
              for (int q = 0; q < 32; ++q) o[q] *= alpha;
              sm100::tmem_st32(tO + 32 * hh, o);
            }
            l *= alpha;
            m = m_new;
          }
        } else {
          m = mx;
        }
        const float nm = -m * sc2;
        if (trw) L2TR(t, c, 4);
        float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // two row-sum chains
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float pk[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int cc = 64 * hh + 2 * q;
            const float2 tt = __ffma2_rn(make_float2(x[cc], x[cc + 1]), make_float2(sc2, sc2), make_float2(nm, nm));
            const float2 ee = make_float2(ex2_approx(tt.x), ex2_approx(tt.y));
            ls[q & 1] = __fadd2_rn(ls[q & 1], ee);
            pk[q] = __uint_as_float(pack_bf16x2(ee.x, ee.y));
          }
          sm100::tmem_st32(tP + 32 * hh, pk);
        }
        if (trw) L2TR(t, c, 5);
        l += (ls[0].x + ls[1].x) + (ls[0].y + ls[1].y);
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&p_ready[t]);
        if (trw) L2TR(t, c, 6);
        ++c;
      }
      pend = true;
      pd_st = st, pd_len = len, pd_h = h, pd_row = q0 + r, pd_m = m, pd_l = l;
    }
    if (pend) readout(pd_st, pd_len, pd_h, pd_row, pd_m, pd_l);
    if (lane == 0) sm100::bulk_wait0();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tbase, 512);
}

// Backward: a software-pipelined persistent kernel.  Warp 8 (one lane) is the producer/issuer:
// TMA loads of (Q, K, V, dO) for the next two units into two smem buffers; S = QK^T and dP = dO V^T
// of unit i+1 as soon as the compute warps have consumed unit i's S/dP; dV = P^T dO of unit i as
// soon as P is in shared memory (while the compute warps form dS), then dK = dS^T Q, dQ = dS K.
// Warps 0-7 do the elementwise softmax-gradient of unit i, then read dV (already done) and dK/dQ
// out of TMEM, so loads, the three MMA batches and the CUDA-core work of neighbouring units overlap.
// TMEM: S [0,128), dP [128,256), dV [256,320), dK [320,384), dQ [384,448).
constexpr int BWD_BUF_BYTES = 4 * TILE_BYTES;  // Q, K, V, dO
constexpr int SH_BWD_THREADS = SH_THREADS + 32;
constexpr int BW_UMAX = 512;  // work units per CTA (build_group_list)
constexpr int SH_BWD_SMEM = 2 * BWD_BUF_BYTES + 2 * P_BYTES + 1024 + 256 + 16 * BW_UMAX;

// per-warp transpose-reduce: lane l ends with sum over the warp's 32 rows of column l of v[32]
__device__ __forceinline__ float warp_colsum32(float* v, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const bool up = lane & s;
      const float send = up ? v[j] : v[j + s];
      const float keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// Backward pass 1 for this thread's 64 keys [64 ch, 64 ch + 64) of query row r:
//   P_rj = 2^(S_rj log2e / sqrt(d) - m_h log2e |r - j| - LSE_r log2e)
// in fp32, written back over S in TMEM (pass 2 reloads it; keeps 64 registers free) and as bf16
// into the swizzled P tile, plus the partial row sum of P * dP (D_r = dO_r . O_r = sum_j P_rj
// dP_rj, so D needs neither O nor dO from memory).  Two keys per instruction on the paired fp32
// pipe; MASK = false for units of exactly 128 rows (no masking).
template <bool MASK>
__device__ __forceinline__ float bwd_pass1(uint32_t tS, uint32_t tdP, uint32_t sPa, int r, int ch, int lo, int hi,
                                          bool row_ok, float sc2, float sl2, float lse2) {
  const uint32_t wwin = (uint32_t)(hi - lo);
  float2 Dp = make_float2(0.f, 0.f);
  const float rc = (float)(r - 64 * ch);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int c0 = 64 * ch + 16 * c;
    float v[16], w[16];
    sm100::tmem_ld16(tS + c0, v);
    sm100::tmem_ld16(tdP + c0, w);
    sm100::tmem_ld_wait();
    uint32_t pp[8];
#pragma unroll
    for (int jj = 0; jj < 16; jj += 2) {
      const float j0 = (float)(16 * c + jj);
      const float2 dd = __fadd2_rn(make_float2(rc, rc), make_float2(-j0, -j0 - 1.f));
      const float2 t = __ffma2_rn(make_float2(fabsf(dd.x), fabsf(dd.y)), make_float2(-sl2, -sl2),
                                  make_float2(-lse2, -lse2));
      const float2 x = __ffma2_rn(make_float2(v[jj], v[jj + 1]), make_float2(sc2, sc2), t);
      float2 pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
      if (MASK) {  // keys outside the row's own sequence, rows past the unit
        pv.x = (row_ok && (uint32_t)(c0 + jj - lo) < wwin) ? pv.x : 0.f;
        pv.y = (row_ok && (uint32_t)(c0 + jj + 1 - lo) < wwin) ? pv.y : 0.f;
      }
      v[jj] = pv.x;
      v[jj + 1] = pv.y;
      Dp = __ffma2_rn(pv, make_float2(w[jj], w[jj + 1]), Dp);
      pp[jj >> 1] = pack_bf16x2(pv.x, pv.y);
    }
    sm100::tmem_st16(tS + c0, v);
    st_shared_v4(sPa + p_off(r, c0), pp[0], pp[1], pp[2], pp[3]);
    st_shared_v4(sPa + p_off(r, c0 + 8), pp[4], pp[5], pp[6], pp[7]);
  }
  sm100::tmem_st_wait();
  return Dp.x + Dp.y;
}

__global__ void __launch_bounds__(SH_BWD_THREADS, 1) attn_bwd_short_kernel(
    const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
    const __grid_constant__ CUtensorMap tm_dqkv, const int* __restrict__ cu,
    int batch, int heads, int d, const float* __restrict__ slopes, const bf16* __restrict__ O,
    const bf16* __restrict__ dO, const float* __restrict__ lse, bf16* __restrict__ dqkv, float* __restrict__ dbias,
    int nnz) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bufs = smem;                        // 2 x (Q, K, V, dO)
  uint8_t* sP = smem + 2 * BWD_BUF_BYTES;
  uint8_t* sdS = sP + P_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + P_BYTES);
  uint64_t* load_full = bars;      // [2]
  uint64_t* sp_full = bars + 2;    // S, dP of the unit in TMEM
  uint64_t* elem_done = bars + 3;  // 8 compute warps: S/dP consumed, dS in smem
  uint64_t* acc_full = bars + 4;   // dK, dQ (and dV) of the unit in TMEM
  uint64_t* p_ready = bars + 5;    // 8 compute warps: P in smem
  uint64_t* dv_full = bars + 6;    // dV of the unit in TMEM
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
  int4* ulist = reinterpret_cast<int4*>(bars + 10);  // this CTA's units (build_group_list)
  __shared__ float dred[2 * 128];  // partial D of the two half-row threads
  __shared__ int wcount[SH_BWD_THREADS / 32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = heads * d;
  if (tid == 0) {
    sm100::tma_prefetch(&tm_qkv);
    sm100::tma_prefetch(&tm_do);
    sm100::tma_prefetch(&tm_dqkv);
    sm100::mbar_init(&load_full[0], 1);
    sm100::mbar_init(&load_full[1], 1);
    sm100::mbar_init(sp_full, 1);
    sm100::mbar_init(elem_done, 8);
    sm100::mbar_init(acc_full, 1);
    sm100::mbar_init(p_ready, 8);
    sm100::mbar_init(dv_full, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();  // (PDL) the setup above touched only shared memory, TMEM and kernel parameters
  pdl_trigger();
  const uint32_t tS = tbase, tdP = tbase + 128, tdV = tbase + 256, tdK = tbase + 320, tdQ = tbase + 384;
  const uint32_t sPa = sm100::smem_u32(sP), sdSa = sm100::smem_u32(sdS);

  const int nunits = build_group_list<SH_BWD_THREADS>(cu, batch, heads, ulist, wcount);

  if (warp == 8) {
    // ------------------------------------------------------------------ producer / MMA issuer
    {  // the whole warp runs the loop: lane 0 issues the TMA loads, one elected lane the MMAs
      auto buf_addr = [&](int b) { return bufs + b * BWD_BUF_BYTES; };
      auto issue_loads = [&](int i, int b) {
        const int4 e = ulist[i];
        const int h = e.z & 0xffff, st = e.x;
        uint8_t* base = buf_addr(b);
        if (lane == 0) {
          sm100::mbar_arrive_expect_tx(&load_full[b], BWD_BUF_BYTES);
          sm100::tma_load_2d(base, &tm_qkv, &load_full[b], h * d, st);
          sm100::tma_load_2d(base + TILE_BYTES, &tm_qkv, &load_full[b], H + h * d, st);
          sm100::tma_load_2d(base + 2 * TILE_BYTES, &tm_qkv, &load_full[b], 2 * H + h * d, st);
          sm100::tma_load_2d(base + 3 * TILE_BYTES, &tm_do, &load_full[b], h * d, st);
        }
        __syncwarp();
      };
      auto mma1 = [&](int b) {  // S = Q K^T, dP = dO V^T
        const uint32_t q = sm100::smem_u32(buf_addr(b));
        const uint32_t k = q + TILE_BYTES, v = q + 2 * TILE_BYTES, o = q + 3 * TILE_BYTES;
        constexpr uint32_t id_s = sm100::idesc_bf16(128, 128, 0, 0);
        for (int kk = 0; kk < d / 16; ++kk) {
          sm100::mma_bf16_ss_w(tS, sm100::desc_kmajor_sw128(q + kk * 32), sm100::desc_kmajor_sw128(k + kk * 32), id_s,
                             kk > 0);
          sm100::mma_bf16_ss_w(tdP, sm100::desc_kmajor_sw128(o + kk * 32), sm100::desc_kmajor_sw128(v + kk * 32), id_s,
                             kk > 0);
        }
        sm100::mma_commit_w(sp_full);
      };
      constexpr uint32_t id_t = sm100::idesc_bf16(128, 64, 1, 1);
      constexpr uint32_t id_q = sm100::idesc_bf16(128, 64, 0, 1);
      auto mma_dv = [&](int b) {  // dV = P^T dO
        const uint32_t o = sm100::smem_u32(buf_addr(b)) + 3 * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          sm100::mma_bf16_ss_w(tdV, sm100::desc_mnmajor_sw128(sPa + kk * 2048, TILE * 128),
                             sm100::desc_mnmajor_sw128(o + kk * 2048, 8192), id_t, kk > 0);
        sm100::mma_commit_w(dv_full);
      };
      auto mma_dkq = [&](int b) {  // dK = dS^T Q, dQ = dS K
        const uint32_t q = sm100::smem_u32(buf_addr(b));
        const uint32_t k = q + TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk) {
          sm100::mma_bf16_ss_w(tdK, sm100::desc_mnmajor_sw128(sdSa + kk * 2048, TILE * 128),
                             sm100::desc_mnmajor_sw128(q + kk * 2048, 8192), id_t, kk > 0);
          sm100::mma_bf16_ss_w(tdQ, sm100::desc_kmajor_sw128(sdSa + (kk >> 2) * (TILE * 128) + (kk & 3) * 32),
                             sm100::desc_mnmajor_sw128(k + kk * 2048, 8192), id_q, kk > 0);
        }
        sm100::mma_commit_w(acc_full);
      };
      if (nunits > 0) issue_loads(0, 0);
      if (nunits > 1) issue_loads(1, 1);
      if (nunits > 0) {
        sm100::mbar_wait(&load_full[0], 0);
        sm100::tc_fence_after();
        mma1(0);
      }
      for (int i = 0; i < nunits; ++i) {
        const int b = i & 1;
        sm100::mbar_wait(p_ready, i & 1);  // P(i) in smem (and dV(i-1) read out)
        sm100::tc_fence_after();
        mma_dv(b);
        sm100::mbar_wait(elem_done, i & 1);  // S/dP(i) consumed, dS(i) in smem
        sm100::tc_fence_after();
        mma_dkq(b);
        if (i + 1 < nunits) {
          sm100::mbar_wait(&load_full[b ^ 1], ((i + 1) >> 1) & 1);
          sm100::tc_fence_after();
          mma1(b ^ 1);
        }
        sm100::mbar_wait(acc_full, i & 1);  // all MMAs of unit i done: buffer b is free
        if (i + 2 < nunits) issue_loads(i + 2, b);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ compute warps 0-7
    const int ch = warp >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float rsd = rsqrtf((float)d);
    const float sc2 = rsd * LOG2E;
    const bool col_ok = 32 * ch < d;
    // this warp's P / dS slabs (rows [32 q4, +32), columns [64 ch, +64)) double as output staging
    const uint32_t slabP = sPa + ch * (TILE * 128) + q4 * 4096, slabS = sdSa + ch * (TILE * 128) + q4 * 4096;
    auto lse_of = [&](int ii) {  // LSE of row r of unit ii, prefetched one unit ahead (scaled at use)
      if (ii >= nunits) return 0.f;
      const int4 e = ulist[ii];
      return r < e.y ? lse[(size_t)(e.z & 0xffff) * nnz + e.x + r] : 0.f;
    };
    float lse_next = lse_of(0);
    for (int i = 0; i < nunits; ++i) {
      const int4 ue = ulist[i];
      const int h = ue.z & 0xffff, span = ue.z >> 16;
      const int start = ue.x;
      const int len = ue.y;  // rows of the unit (the whole group)
      int lo, hi;
      group_window(ue, r, lo, hi);
      const float sl2 = slopes[h] * LOG2E;
      const float lse2 = lse_next * LOG2E;
      // the previous unit's TMA stores must have read this warp's slabs before they are rewritten
      if (lane == 0) sm100::bulk_wait_read0();
      __syncwarp();
      sm100::mbar_wait(sp_full, i & 1);
      sm100::tc_fence_after();
      const float Dp = (len == TILE && span == 1)
                           ? bwd_pass1<false>(tS + lane_off, tdP + lane_off, sPa, r, ch, 0, TILE, true, sc2, sl2, lse2)
                           : bwd_pass1<true>(tS + lane_off, tdP + lane_off, sPa, r, ch, lo, hi, r < len, sc2, sl2, lse2);
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(p_ready);
      dred[ch * 128 + r] = Dp;
      named_bar_sync(1 + (warp & 3), 64);  // the two half-row warps only
      const float Dr = dred[r] + dred[128 + r];
      // pass 2: dS/sqrt(d) = P (dP - D)/sqrt(d) — the 1/sqrt(d) of dQ = dS K / sqrt(d) and
      // dK = dS^T Q / sqrt(d) is folded in here (exact for d = 64), so the readout does no scaling
      const float Drs = -Dr * rsd;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int c0 = 64 * ch + 32 * c;
        float w[32], pf[32];
        sm100::tmem_ld32(tS + lane_off + c0, pf);  // fp32 P from pass 1
        sm100::tmem_ld32(tdP + lane_off + c0, w);
        sm100::tmem_ld_wait();
        uint32_t pd[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
          const float2 ds = __fmul2_rn(make_float2(pf[jj], pf[jj + 1]),
                                       __ffma2_rn(make_float2(w[jj], w[jj + 1]), make_float2(rsd, rsd),
                                                  make_float2(Drs, Drs)));
          pd[jj >> 1] = pack_bf16x2(ds.x, ds.y);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_shared_v4(sdSa + p_off(r, c0 + q * 8), pd[4 * q], pd[4 * q + 1], pd[4 * q + 2], pd[4 * q + 3]);
      }
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(elem_done);
      lse_next = lse_of(i + 1);  // in flight while the MMAs run
      // dV (row = key r), then dQ (row = query r), dK (row = key r): this thread's 32 of the 64
      // columns.  A warp whose 32 rows all lie inside the sequence stages its [32 x 32] bf16 block
      // in its own P / dS slab (64-byte swizzle, conflict-free) and one lane TMA-stores it; the
      // ragged last quarter of a short sequence stores its valid rows directly.
      const bool ok = r < len;
      const bool full = q4 * 32 + 32 <= len;  // warp-uniform
      sm100::mbar_wait(dv_full, i & 1);
#pragma unroll 1
      for (int k3 = 0; k3 < 3; ++k3) {
        const int which = k3 == 0 ? 2 : k3 - 1;  // V, Q, K
        if (k3 == 1) sm100::mbar_wait(acc_full, i & 1);
        sm100::tc_fence_after();
        float v[32];
        const uint32_t src = which == 0 ? tdQ : (which == 1 ? tdK : tdV);
        sm100::tmem_ld32(src + lane_off + 32 * ch, v);
        sm100::tmem_ld_wait();
        if (!full) {  // rows past the sequence hold garbage accumulations: zero them for the column sums
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = ok ? v[e] : 0.f;
        }
        if (col_ok) {
          if (full) {
            // staging: dV -> P slab [0, 2K) (P was consumed by dV's MMA), dQ -> P slab [2K, 4K),
            // dK -> dS slab (all MMAs done once acc_full has been waited)
            const uint32_t stg = which == 2 ? slabP : (which == 0 ? slabP + 2048 : slabS);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint4 pk = f32_to_bf16x8(v + 8 * c);
              st_shared_v4(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), pk.x, pk.y, pk.z, pk.w);
            }
            sm100::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              sm100::tma_store_2d(&tm_dqkv, stg, which * H + h * d + 32 * ch, start + q4 * 32);
              sm100::bulk_commit();
            }
          } else if (ok) {
            bf16* dst = dqkv + (size_t)(start + r) * 3 * H + which * H + h * d + 32 * ch;
#pragma unroll
            for (int c = 0; c < 32; c += 8) *reinterpret_cast<uint4*>(dst + c) = f32_to_bf16x8(v + c);
          }
        }
        // QKV-projection bias gradient = column sums of dQKV: transpose-reduce over the warp's 32
        // rows, one atomic per column per warp.  The K part is identically zero (R31: a key bias
        // adds q_i.b_k/sqrt(d) to every score of row i, which the row softmax cancels), so it is
        // neither summed nor added.
        if (dbias && which != 1) {
          const float cs = warp_colsum32(v, lane);
          if (col_ok && 32 * ch + lane < d) atomicAdd(dbias + which * H + h * d + 32 * ch + lane, cs);
        }
      }
      sm100::tc_fence_before();
    }
    if (lane == 0) sm100::bulk_wait0();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// Long-sequence backward (128 < l <= 2048): one work unit = (128-key tile j, head, sequence),
// iterating over the sequence's query tiles i.  D_i = dO_i . O_i comes from a pre-pass
// (attn_bwd_prep_kernel), so each (i, j) block needs a single pass over S and dP:
//   P = 2^(S log2e/sqrt(d) - m log2e |q - k| - LSE log2e),  dS/sqrt(d) = P (dP - D)/sqrt(d)
//   dV_j += P^T dO_i, dK_j += dS^T Q_i  (TMEM accumulators across the unit's query tiles)
//   dQ_i += dS K_j                        (per block, folded into an fp32 [nnz, H] buffer by
//                                          TMA bulk reduce-adds; dq_finish_kernel converts it)
// Warp 13 streams K/V (double-buffered per unit) and Q/dO tiles (LB_NS-stage ring) by TMA; warp 12
// issues S, dP of block i+1 as soon as the compute warps 0-7 hold block i's in registers, and
// dV/dK/dQ of block i once P_i, dS_i are in smem; the epilogue warps 8-11 read dQ_i (and, at a
// unit end, dV / dK) out of TMEM and hand them to TMA.  TMEM: S [0,128), dP [128,256),
// dV [256,320), dK [320,384), dQ [384,512) (two buffers).
// ------------------------------------------------------------------------------------------
constexpr int LB_NS = 2;
constexpr int LB_THREADS = SH_THREADS + 256;  // compute warps 0-7; epilogue warps 8-11; MMA warp 12, TMA warp 13
constexpr int LB_SMEM = 2 * 2 * TILE_BYTES + LB_NS * 2 * TILE_BYTES + 3 * P_BYTES + 1024 + 256;  // P + 2 x dS

// D[h, t] = sum_c dO[t, h d + c] O[t, h d + c]  (the rowsum(dO o O) of FlashAttention's backward).
// One warp per token row: lane l reads the row's 16-byte chunks l, l + 32, ... (coalesced 512 B per
// instruction, every load issued before the first use), the d / 8 chunks of a head are reduced
// across their lanes with shuffles.
__global__ void attn_bwd_prep_kernel(const bf16* __restrict__ O, const bf16* __restrict__ dO, int nnz, int heads,
                                     int d, float* __restrict__ D) {
  const int lane = threadIdx.x & 31;
  const int H = heads * d, nch = H / 8, cph = d / 8;  // 16-byte chunks per row / per head
  const int wpb = blockDim.x >> 5;
  for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < nnz; t += gridDim.x * wpb) {
    const bf16* o = O + (size_t)t * H;
    const bf16* g = dO + (size_t)t * H;
    uint4 a[4], b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = lane + 32 * k;
      if (i < nch) {
        a[k] = ld_nc_v4(o + 8 * i);
        b[k] = ld_nc_v4(g + 8 * i);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = lane + 32 * k;
      if (32 * k >= nch) break;  // warp-uniform
      float acc = 0.f;
      if (i < nch) {
        float fa[8], fb[8];
        bf16x8_to_f32(a[k], fa);
        bf16x8_to_f32(b[k], fb);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(fa[e], fb[e], acc);
      }
      for (int m = 1; m < cph; m <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);  // cph | 32: groups align
      if (i < nch && (i % cph) == 0) D[(size_t)(i / cph) * nnz + t] = acc;
    }
  }
}

// dq_acc fp32 [nnz, H] -> dqkv[:, :H] bf16, and db_q += column sums: a CTA of DQF_GROUPS row groups x
// (H / 8) column vectors covers rows_per rows, reduces its groups through smem and issues one
// atomic per column (a few hundred per address instead of one per 16 rows)
constexpr int DQF_GROUPS = 8;
__global__ void dq_finish_kernel(const float* __restrict__ dq_acc, int nnz, int H, int rows_per, bf16* __restrict__ dqkv,
                                 float* __restrict__ db) {
  extern __shared__ float red[];  // [DQF_GROUPS][H]
  const int cv = threadIdx.x, rg = threadIdx.y;
  const int c = cv * 8;
  const int r0 = blockIdx.x * rows_per, r1 = min(nnz, r0 + rows_per);
  float cs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  constexpr int U = 4;  // rows in flight per thread: all loads issued before the first conversion
  for (int rb = r0 + rg; rb < r1; rb += U * DQF_GROUPS) {
    float4 a[U], b[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int r = rb + k * DQF_GROUPS;
      if (r < r1) {
        const float4* src = reinterpret_cast<const float4*>(dq_acc + (size_t)r * H + c);
        a[k] = __ldcs(src);
        b[k] = __ldcs(src + 1);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int r = rb + k * DQF_GROUPS;
      if (r >= r1) break;
      const float t[8] = {a[k].x, a[k].y, a[k].z, a[k].w, b[k].x, b[k].y, b[k].z, b[k].w};
      const uint4 pk = f32_to_bf16x8(t);
      *reinterpret_cast<uint4*>(dqkv + (size_t)r * 3 * H + c) = pk;
      float f[8];
      bf16x8_to_f32(pk, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) cs[e] += f[e];
    }
  }
  if (!db) return;
#pragma unroll
  for (int e = 0; e < 8; ++e) red[rg * H + c + e] = cs[e];
  __syncthreads();
  if (rg == 0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float t = 0.f;
#pragma unroll
      for (int k = 0; k < DQF_GROUPS; ++k) t += red[k * H + c + e];
      atomicAdd(db + c + e, t);
    }
  }
}

// deterministic mode: dQ row r = sum over the key tiles kt < ceil(len_b / 128) of its sequence b of
// slab kt, in kt order; written as bf16 into the Q third of dqkv (db_q then comes from colsum_det)
__global__ void dq_finish_det_kernel(const float* __restrict__ dq_part, const int* __restrict__ cu, int batch, int nnz,
                                     int H, bf16* __restrict__ dqkv) {
  const int r = blockIdx.x * blockDim.y + threadIdx.y;
  const int c = threadIdx.x * 8;
  if (r >= nnz || c >= H) return;
  int lo = 0, hi = batch;  // sequence b with cu[b] <= r < cu[b + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cu[mid] <= r) lo = mid;
    else hi = mid;
  }
  const int nt = (cu[lo + 1] - cu[lo] + TILE - 1) / TILE;
  float t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int kt = 0; kt < nt; ++kt) {
    const float4* src = reinterpret_cast<const float4*>(dq_part + ((size_t)kt * nnz + r) * H + c);
    const float4 a = src[0], b = src[1];
    t[0] += a.x, t[1] += a.y, t[2] += a.z, t[3] += a.w, t[4] += b.x, t[5] += b.y, t[6] += b.z, t[7] += b.w;
  }
  *reinterpret_cast<uint4*>(dqkv + (size_t)r * 3 * H + c) = f32_to_bf16x8(t);
}

// single-pass P / dS of one (q tile, k tile) block for this thread's 64 keys: P -> sP as computed;
// dS/sqrt(d) is kept packed in registers and written to sdS after this warp's pending bulk copies
// (the previous block's dQ reduction staged in the dS slab) have read it
template <bool MASK>
__device__ __forceinline__ void bwd_block(uint32_t tS, uint32_t tdP, uint32_t sPa, uint32_t sdSa, int r, int ch,
                                          int lane, int qk_off, int qrows, int keys, float sc2, float sl2, float lse2,
                                          float rsd, float Drs) {
  const float rc = (float)(r + qk_off - 64 * ch);
  uint32_t pd[32];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int c0 = 64 * ch + 16 * c;
    float v[16], w[16];
    sm100::tmem_ld16(tS + c0, v);
    sm100::tmem_ld16(tdP + c0, w);
    sm100::tmem_ld_wait();
    uint32_t pp[8];
#pragma unroll
    for (int jj = 0; jj < 16; jj += 2) {
      const float j0 = (float)(16 * c + jj);
      const float2 dd = __fadd2_rn(make_float2(rc, rc), make_float2(-j0, -j0 - 1.f));
      const float2 t = __ffma2_rn(make_float2(fabsf(dd.x), fabsf(dd.y)), make_float2(-sl2, -sl2),
                                  make_float2(-lse2, -lse2));
      const float2 x = __ffma2_rn(make_float2(v[jj], v[jj + 1]), make_float2(sc2, sc2), t);
      float2 pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
      if (MASK) {
        pv.x = (r < qrows && c0 + jj < keys) ? pv.x : 0.f;
        pv.y = (r < qrows && c0 + jj + 1 < keys) ? pv.y : 0.f;
      }
      const float2 ds = __fmul2_rn(pv, __ffma2_rn(make_float2(w[jj], w[jj + 1]), make_float2(rsd, rsd),
                                                  make_float2(Drs, Drs)));
      pp[jj >> 1] = pack_bf16x2(pv.x, pv.y);
      pd[8 * c + (jj >> 1)] = pack_bf16x2(ds.x, ds.y);
    }
    st_shared_v4(sPa + p_off(r, c0), pp[0], pp[1], pp[2], pp[3]);
    st_shared_v4(sPa + p_off(r, c0 + 8), pp[4], pp[5], pp[6], pp[7]);
  }
  if (lane == 0) sm100::bulk_wait_read0();
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(sdSa + p_off(r, 64 * ch + 8 * c), pd[4 * c], pd[4 * c + 1], pd[4 * c + 2], pd[4 * c + 3]);
}

// the same block computation from S / dP already in registers (v = S, w = dP: this thread's 64 keys)
template <bool MASK>
__device__ __forceinline__ void bwd_block_regs(const float (&v)[64], const float (&w)[64], uint32_t sPa, uint32_t sdSa,
                                               int r, int ch, int lane, int qk_off, int qrows, int keys, float sc2,
                                               float sl2, float lse2, float rsd, float Drs) {
  const float rc = (float)(r + qk_off - 64 * ch);
  uint32_t pd[32];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int c0 = 64 * ch + 16 * c;
    uint32_t pp[8];
#pragma unroll
    for (int jj = 0; jj < 16; jj += 2) {
      const int j = 16 * c + jj;
      const float2 dd = __fadd2_rn(make_float2(rc, rc), make_float2(-(float)j, -(float)j - 1.f));
      const float2 t = __ffma2_rn(make_float2(fabsf(dd.x), fabsf(dd.y)), make_float2(-sl2, -sl2),
                                  make_float2(-lse2, -lse2));
      const float2 x = __ffma2_rn(make_float2(v[j], v[j + 1]), make_float2(sc2, sc2), t);
      float2 pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
      if (MASK) {
        pv.x = (r < qrows && c0 + jj < keys) ? pv.x : 0.f;
        pv.y = (r < qrows && c0 + jj + 1 < keys) ? pv.y : 0.f;
      }
      const float2 ds = __fmul2_rn(pv, __ffma2_rn(make_float2(w[j], w[j + 1]), make_float2(rsd, rsd),
                                                  make_float2(Drs, Drs)));
      pp[jj >> 1] = pack_bf16x2(pv.x, pv.y);
      pd[8 * c + (jj >> 1)] = pack_bf16x2(ds.x, ds.y);
    }
    st_shared_v4(sPa + p_off(r, c0), pp[0], pp[1], pp[2], pp[3]);
    st_shared_v4(sPa + p_off(r, c0 + 8), pp[4], pp[5], pp[6], pp[7]);
  }
  if (lane == 0) sm100::bulk_wait_read0();
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(sdSa + p_off(r, 64 * ch + 8 * c), pd[4 * c], pd[4 * c + 1], pd[4 * c + 2], pd[4 * c + 3]);
}

__global__ void __launch_bounds__(LB_THREADS, 1) attn_bwd_long_kernel(
    const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
    const __grid_constant__ CUtensorMap tm_dqkv, const __grid_constant__ CUtensorMap tm_dq, LongUnits U, int d,
    const float* __restrict__ slopes,
    const float* __restrict__ lse, const float* __restrict__ Dg, float* __restrict__ dq_acc,
    bf16* __restrict__ dqkv, float* __restrict__ dbias, int nnz, int det) {
  // det (deterministic mode): each key tile kt stores its dQ contribution into its own slab
  // dq_acc[kt * nnz + row] (tm_dq spans [QT * nnz, H]) instead of reduce-adding into one buffer;
  // dq_finish_det_kernel then sums the slabs in key-tile order
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sKV = smem;                           // 2 x (K, V)
  uint8_t* sQD = sKV + 2 * 2 * TILE_BYTES;       // LB_NS x (Q, dO)
  uint8_t* sP = sQD + LB_NS * 2 * TILE_BYTES;
  uint8_t* sdS = sP + P_BYTES;                   // 2 x dS: block g uses buffer g & 1, then stages its outputs
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + 2 * P_BYTES);
  uint64_t* kv_full = bars;                      // [2]
  uint64_t* kv_empty = bars + 2;                 // [2]
  uint64_t* qd_full = bars + 4;                  // [LB_NS]
  uint64_t* qd_empty = bars + 4 + LB_NS;         // [LB_NS]
  uint64_t* sp_full = bars + 4 + 2 * LB_NS;
  uint64_t* elem_done = sp_full + 1;             // 8 compute warps: P_g, dS_g in smem
  uint64_t* out_free = sp_full + 2;              // 4 epilogue warps: the unit's dV / dK are out of TMEM
  uint64_t* sp_free = sp_full + 3;               // 8 compute warps: S / dP of the block are in registers
  uint64_t* p_free = sp_full + 4;                // dV MMAs of the block done: P may be overwritten
  // per buffer b = g & 1 (a single acc_full could run two phases ahead of the decoupled epilogue):
  uint64_t* acc_full = sp_full + 5;              // [2] block g's MMAs complete (dQ_g; dV / dK at a unit end)
  uint64_t* ds_free = sp_full + 7;               // [2] 4 epilogue warps: dS buffer b free (its staging read)
  uint64_t* dq_free = sp_full + 9;               // [2] 4 epilogue warps: dQ TMEM buffer b read out
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sp_full + 11);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = U.heads * d;
  if (tid == 0) {
    sm100::tma_prefetch(&tm_qkv);
    sm100::tma_prefetch(&tm_do);
    sm100::tma_prefetch(&tm_dqkv);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
      sm100::mbar_init(&ds_free[i], 4);
      sm100::mbar_init(&dq_free[i], 4);
      sm100::mbar_init(&acc_full[i], 1);
    }
    for (int i = 0; i < LB_NS; ++i) {
      sm100::mbar_init(&qd_full[i], 1);
      sm100::mbar_init(&qd_empty[i], 1);
    }
    sm100::mbar_init(sp_full, 1);
    sm100::mbar_init(elem_done, 8);
    sm100::mbar_init(out_free, 4);
    sm100::mbar_init(sp_free, 8);
    sm100::mbar_init(p_free, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();  // (PDL) the setup above touched only shared memory, TMEM and kernel parameters
  pdl_trigger();
  // dQ is double-buffered in TMEM (block g accumulates into tdQ + 64 (g & 1)) so the epilogue
  // warpgroup reads it out while the next block's MMAs run
  const uint32_t tS = tbase, tdP = tbase + 128, tdV = tbase + 256, tdK = tbase + 320, tdQ = tbase + 384;
  const uint32_t sKVa = sm100::smem_u32(sKV), sQDa = sm100::smem_u32(sQD), sPa = sm100::smem_u32(sP),
                 sdSa = sm100::smem_u32(sdS);
  auto nq_of = [&](int u) {
    int b, h, jt;
    U.decode(u, b, h, jt);
    return (U.cu[b + 1] - U.cu[b] + TILE - 1) / TILE;
  };

  // registers: 16 warps leave 128 per thread; the compute warpgroups (S and dP rows in registers)
  // take 192, the epilogue warpgroup 88 and the producer / issuer warpgroup 40
  if (warp >= 12) {
    sm100::setmaxnreg_dec<40>();
    if (warp == 13) {
      // ---------------------------------------------------------------- TMA producer
      if (lane == 0) {
        int uc = 0, g = 0;
        for (int u = U.first(); u < U.total; u = U.next(u), ++uc) {
          int b, h, jt;
          U.decode(u, b, h, jt);
          const int st = U.cu[b], nq = (U.cu[b + 1] - st + TILE - 1) / TILE;
          const int kb = uc & 1;
          sm100::mbar_wait(&kv_empty[kb], ((uc >> 1) & 1) ^ 1);
          uint8_t* kv = sKV + kb * 2 * TILE_BYTES;
          sm100::mbar_arrive_expect_tx(&kv_full[kb], 2 * TILE_BYTES);
          sm100::tma_load_2d(kv, &tm_qkv, &kv_full[kb], H + h * d, st + jt * TILE);
          sm100::tma_load_2d(kv + TILE_BYTES, &tm_qkv, &kv_full[kb], 2 * H + h * d, st + jt * TILE);
          for (int i = 0; i < nq; ++i, ++g) {
            const int sg = g % LB_NS;
            sm100::mbar_wait(&qd_empty[sg], ((g / LB_NS) & 1) ^ 1);
            uint8_t* qd = sQD + sg * 2 * TILE_BYTES;
            sm100::mbar_arrive_expect_tx(&qd_full[sg], 2 * TILE_BYTES);
            sm100::tma_load_2d(qd, &tm_qkv, &qd_full[sg], h * d, st + i * TILE);
            sm100::tma_load_2d(qd + TILE_BYTES, &tm_do, &qd_full[sg], h * d, st + i * TILE);
          }
        }
      }
      __syncwarp();
    } else if (warp == 12) {
      // ---------------------------------------------------------------- MMA issuer (whole warp, elected lane)
      constexpr uint32_t id_s = sm100::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_t = sm100::idesc_bf16(128, 64, 1, 1);  // P^T dO, dS^T Q
      constexpr uint32_t id_q = sm100::idesc_bf16(128, 64, 0, 1);  // dS K
      int u = U.first(), uc = 0, i = 0, nq = u < U.total ? nq_of(u) : 0;
      auto mma1 = [&](int g, int ucc) {  // S = Q_i K_j^T, dP = dO_i V_j^T
        const int sg = g % LB_NS;
        sm100::mbar_wait(&qd_full[sg], (g / LB_NS) & 1);
        sm100::tc_fence_after();
        const uint32_t q = sQDa + sg * 2 * TILE_BYTES, o = q + TILE_BYTES;
        const uint32_t k = sKVa + (ucc & 1) * 2 * TILE_BYTES, v = k + TILE_BYTES;
        for (int kk = 0; kk < d / 16; ++kk) {
          sm100::mma_bf16_ss_w(tS, sm100::desc_kmajor_sw128(q + kk * 32), sm100::desc_kmajor_sw128(k + kk * 32), id_s,
                               kk > 0);
          sm100::mma_bf16_ss_w(tdP, sm100::desc_kmajor_sw128(o + kk * 32), sm100::desc_kmajor_sw128(v + kk * 32), id_s,
                               kk > 0);
        }
        sm100::mma_commit_w(sp_full);
      };
      if (u < U.total) {
        sm100::mbar_wait(&kv_full[0], 0);
        mma1(0, 0);
      }
      for (int g = 0; u < U.total; ++g) {
        // cursor of block g + 1; its S / dP go into TMEM as soon as block g's are in registers
        int u2 = u, uc2 = uc, i2 = i + 1, nq2 = nq;
        if (i2 == nq) {
          u2 = U.next(u);
          ++uc2;
          i2 = 0;
          nq2 = u2 < U.total ? nq_of(u2) : 0;
        }
        sm100::mbar_wait(sp_free, g & 1);
        if (u2 < U.total) {
          if (i2 == 0) sm100::mbar_wait(&kv_full[uc2 & 1], (uc2 >> 1) & 1);
          mma1(g + 1, uc2);
        }
        sm100::mbar_wait(elem_done, g & 1);                               // P_g, dS_g in smem
        if (i == 0 && uc > 0) sm100::mbar_wait(out_free, (uc - 1) & 1);  // previous unit's dV / dK read out
        sm100::tc_fence_after();
        const int sg = g % LB_NS;
        const uint32_t q = sQDa + sg * 2 * TILE_BYTES, o = q + TILE_BYTES;
        const uint32_t k = sKVa + (uc & 1) * 2 * TILE_BYTES;
        const uint32_t ds = sdSa + (g & 1) * P_BYTES, dq = tdQ + (g & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          sm100::mma_bf16_ss_w(tdV, sm100::desc_mnmajor_sw128(sPa + kk * 2048, TILE * 128),
                               sm100::desc_mnmajor_sw128(o + kk * 2048, 8192), id_t, (i > 0 || kk > 0) ? 1u : 0u);
        sm100::mma_commit_w(p_free);  // P of block g + 1 may be written while dK / dQ of block g run
        if (g >= 2) {                 // the epilogue has read dQ of block g - 2 out of this TMEM buffer
          sm100::mbar_wait(&dq_free[g & 1], ((g >> 1) - 1) & 1);
          sm100::tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk) {
          sm100::mma_bf16_ss_w(tdK, sm100::desc_mnmajor_sw128(ds + kk * 2048, TILE * 128),
                               sm100::desc_mnmajor_sw128(q + kk * 2048, 8192), id_t, (i > 0 || kk > 0) ? 1u : 0u);
          sm100::mma_bf16_ss_w(dq, sm100::desc_kmajor_sw128(ds + (kk >> 2) * (TILE * 128) + (kk & 3) * 32),
                               sm100::desc_mnmajor_sw128(k + kk * 2048, 8192), id_q, kk > 0);
        }
        sm100::mma_commit_w(&acc_full[g & 1]);
        sm100::mma_commit_w(&qd_empty[sg]);
        if (i2 == 0) sm100::mma_commit_w(&kv_empty[uc & 1]);  // the unit's last read of K_j, V_j
        u = u2, uc = uc2, i = i2, nq = nq2;
      }
    }
    __syncwarp();
  } else if (warp >= 8) {
    // ------------------------------------------------------------------ epilogue warps 8-11
    // Per block: dQ_g out of TMEM, staged as fp32 in this warp's quarter of dS buffer g & 1 (free once
    // block g's MMAs are), handed to the TMA engine as a bulk reduce-add (det: a store into slab kt).
    // Per unit end: dV, dK out of TMEM (then out_free), staged as bf16 in the same quarter, TMA stores.
    // The quarter is released (ds_free) once the bulk copies have read it.
    sm100::setmaxnreg_dec<88>();
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int g = 0;
    for (int u = U.first(); u < U.total; u = U.next(u)) {
      int b, h, jt;
      U.decode(u, b, h, jt);
      const int start = U.cu[b], len = U.cu[b + 1] - start, kv0 = jt * TILE;
      const int nq = (len + TILE - 1) / TILE;
      for (int i = 0; i < nq; ++i, ++g) {
        const int q0 = i * TILE;
        const uint32_t stg = sdSa + (g & 1) * P_BYTES + q4 * 8192;  // 8 KB: two [32 x 32] fp32 blocks
        sm100::mbar_wait(&acc_full[g & 1], (g >> 1) & 1);
        sm100::tc_fence_after();
        const bool full_rows = q0 + q4 * 32 + 32 <= len;  // warp-uniform
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          float v[32];
          sm100::tmem_ld32(tdQ + (g & 1) * 64 + lane_off + 32 * hh, v);
          sm100::tmem_ld_wait();
          if (hh == 1) {
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&dq_free[g & 1]);
          }
          if (32 * hh >= d) continue;
          if (full_rows) {
            const uint32_t blk = stg + hh * 4096;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              st_shared_v4(blk + lane * 128 + ((c ^ (lane & 7)) << 4), __float_as_uint(v[4 * c]),
                           __float_as_uint(v[4 * c + 1]), __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3]));
            sm100::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (det) sm100::tma_store_2d(&tm_dq, blk, h * d + 32 * hh, jt * nnz + start + q0 + q4 * 32);
              else sm100::tma_reduce_add_2d(&tm_dq, blk, h * d + 32 * hh, start + q0 + q4 * 32);
              sm100::bulk_commit();
            }
          } else if (q0 + r < len) {
            float* dst = dq_acc + ((size_t)(det ? jt * nnz : 0) + start + q0 + r) * H + h * d + 32 * hh;
            if (det) {
#pragma unroll
              for (int e = 0; e < 32; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 32; e += 4) red_add_v4(dst + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
          }
        }
        if (i + 1 == nq) {
          // unit end: dV / dK of the key tile (rows = keys kv0 + r), final with block g's MMAs
          const bool ok = kv0 + r < len;
          const bool full = kv0 + q4 * 32 + 32 <= len;  // warp-uniform
          if (lane == 0) sm100::bulk_wait_read0();      // the dQ blocks have left the staging quarter
          __syncwarp();
#pragma unroll 1
          for (int w4 = 0; w4 < 4; ++w4) {  // (V, K) x (columns 0-31, 32-63)
            const int which = w4 < 2 ? 2 : 1, hh = w4 & 1;
            float v[32];
            sm100::tmem_ld32((which == 2 ? tdV : tdK) + lane_off + 32 * hh, v);
            sm100::tmem_ld_wait();
            if (w4 == 3) {
              sm100::tc_fence_before();
              __syncwarp();
              if (lane == 0) sm100::mbar_arrive(out_free);
            }
            if (!full) {
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = ok ? v[e] : 0.f;
            }
            const bool col_ok = 32 * hh < d;
            if (col_ok) {
              if (full) {
                const uint32_t blk = stg + w4 * 2048;  // [32 x 32] bf16, 64B swizzle
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const uint4 pk = f32_to_bf16x8(v + 8 * c);
                  st_shared_v4(blk + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), pk.x, pk.y, pk.z, pk.w);
                }
                sm100::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  sm100::tma_store_2d(&tm_dqkv, blk, which * H + h * d + 32 * hh, start + kv0 + q4 * 32);
                  sm100::bulk_commit();
                }
              } else if (ok) {
                bf16* dst = dqkv + (size_t)(start + kv0 + r) * 3 * H + which * H + h * d + 32 * hh;
#pragma unroll
                for (int c = 0; c < 32; c += 8) *reinterpret_cast<uint4*>(dst + c) = f32_to_bf16x8(v + c);
              }
            }
            if (dbias && which == 2) {  // db_v = column sums of dV (db_k = 0, R31; db_q in dq_finish_kernel)
              const float cs = warp_colsum32(v, lane);
              if (col_ok && 32 * hh + lane < d) atomicAdd(dbias + 2 * H + h * d + 32 * hh + lane, cs);
            }
          }
        }
        // the staging quarter of dS buffer g & 1 is free once the bulk copies have read it
        if (lane == 0) sm100::bulk_wait_read0();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&ds_free[g & 1]);
      }
    }
    if (lane == 0) sm100::bulk_wait0();
  } else {
    // ------------------------------------------------------------------ compute warps 0-7
    sm100::setmaxnreg_inc<192>();  // 8 x 32 x 192 + 4 x 32 x 88 + 4 x 32 x 40 <= 16 x 32 x 128
    const int ch = warp >> 2, q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const float rsd = rsqrtf((float)d);
    const float sc2 = rsd * LOG2E;
    int g = 0;
    // LSE and D of row r of query tile ii of unit uu, loaded one block ahead of their use
    auto row_stats = [&](int uu, int ii, float& l_, float& d_) {
      l_ = 0.f, d_ = 0.f;
      if (uu >= U.total) return;
      int bb, hh, jj;
      U.decode(uu, bb, hh, jj);
      const int st = U.cu[bb], q = ii * TILE + r;
      if (q < U.cu[bb + 1] - st) {
        l_ = lse[(size_t)hh * nnz + st + q];
        d_ = Dg[(size_t)hh * nnz + st + q];
      }
    };
    float lse_c, D_c;
    row_stats(U.first(), 0, lse_c, D_c);
    for (int u = U.first(); u < U.total; u = U.next(u)) {
      int b, h, jt;
      U.decode(u, b, h, jt);
      const int start = U.cu[b], len = U.cu[b + 1] - start, kv0 = jt * TILE;
      const int nq = (len + TILE - 1) / TILE;
      const float sl2 = slopes[h] * LOG2E;
      const int un = U.next(u);
      for (int i = 0; i < nq; ++i, ++g) {
        const int q0 = i * TILE;
        const float lse2 = lse_c * LOG2E;
        const float Drs = -D_c * rsd;
        if (i + 1 < nq) row_stats(u, i + 1, lse_c, D_c);
        else row_stats(un, 0, lse_c, D_c);
        sm100::mbar_wait(sp_full, g & 1);
        sm100::tc_fence_after();
        float sv[64], dpv[64];
        sm100::tmem_ld32(tS + lane_off + 64 * ch, sv);
        sm100::tmem_ld32(tS + lane_off + 64 * ch + 32, sv + 32);
        sm100::tmem_ld32(tdP + lane_off + 64 * ch, dpv);
        sm100::tmem_ld32(tdP + lane_off + 64 * ch + 32, dpv + 32);
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(sp_free);  // S / dP of the next block may overwrite TMEM
        // P is single-buffered: block g-1's dV MMAs must have read it; dS buffer g & 1 was last used by
        // block g-2, whose MMAs and output staging the epilogue has finished with
        if (g > 0) sm100::mbar_wait(p_free, (g - 1) & 1);
        if (g >= 2) sm100::mbar_wait(&ds_free[g & 1], ((g >> 1) - 1) & 1);
        const uint32_t sdSg = sdSa + (g & 1) * P_BYTES;
        if (len - q0 >= TILE && len - kv0 >= TILE)
          bwd_block_regs<false>(sv, dpv, sPa, sdSg, r, ch, lane, q0 - kv0, len - q0, len - kv0, sc2, sl2, lse2, rsd,
                                Drs);
        else
          bwd_block_regs<true>(sv, dpv, sPa, sdSg, r, ch, lane, q0 - kv0, len - q0, len - kv0, sc2, sl2, lse2, rsd,
                               Drs);
        sm100::fence_proxy_async_smem();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(elem_done);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 0) sm100::tmem_dealloc(tbase, 512);
}

}  // namespace

mb_status attention_fwd(const bf16* qkv, const int* cu, int batch, int nnz, int max_seqlen, int heads, int d,
                        const float* slopes, bf16* O, float* lse, cudaStream_t s) {
  if (nnz == 0 || batch == 0) return MB_OK;
  MB_REQUIRE(d == 32 || d == 64, MB_ERR_CONFIG);
  MB_REQUIRE(max_seqlen >= 1 && max_seqlen <= kMaxSeqlen, MB_ERR_SHAPE);
  const int H = heads * d;
  CUtensorMap tm;
  MB_REQUIRE(make_tmap_bf16_2d(&tm, qkv, 3 * H, nnz, 3 * H, DT, TILE), MB_ERR_CUDA);
  static const bool short_v1 = [] {  // MB_ATTN_SHORT_FWD=v1: the round-1 short kernel (A/B)
    const char* e = std::getenv("MB_ATTN_SHORT_FWD");
    return e && e[0] == 'v' && e[1] == '1';
  }();
  if (max_seqlen <= TILE && !short_v1) {
    static bool attr_s2 = false;
    if (!attr_s2) {
      if (cudaFuncSetAttribute(attn_fwd_short2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, S2_SMEM) !=
          cudaSuccess)
        return MB_ERR_CUDA;
      attr_s2 = true;
    }
    CUtensorMap tmo2;  // [32 rows x 32 columns] output blocks, 64-byte swizzle
    MB_REQUIRE(make_tmap_bf16_2d(&tmo2, O, H, nnz, H, 32, 32, 64), MB_ERR_CUDA);
    // a CTA's unit list holds S2_UMAX units: larger batches go in chunks of sequences (cu_seqlens
    // holds absolute token offsets, so a chunk is just an offset into it)
    const int chunk = std::max(1, num_sms() * S2_UMAX / heads);
    for (int b0 = 0; b0 < batch; b0 += chunk) {
      const int nb = std::min(chunk, batch - b0);
      const int grid = std::max(1, std::min(nb * heads, num_sms()));
      if (launch_pdl(attn_fwd_short2_kernel, dim3(grid), dim3(S2_THREADS), S2_SMEM, s, 1, tm, tmo2, cu + b0, nb, heads,
                     d, slopes, O, lse, nnz) != cudaSuccess)
        return MB_ERR_CUDA;
      MB_CHECK_LAUNCH();
    }
    return MB_OK;
  }
  if (max_seqlen <= TILE) {
    static bool attr_s = false;
    if (!attr_s) {
      if (cudaFuncSetAttribute(attn_fwd_short_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SH_FWD_SMEM2) !=
          cudaSuccess)
        return MB_ERR_CUDA;
      attr_s = true;
    }
    CUtensorMap tmo;  // [32 rows x 32 columns] output blocks, 64-byte swizzle
    MB_REQUIRE(make_tmap_bf16_2d(&tmo, O, H, nnz, H, 32, 32, 64), MB_ERR_CUDA);
    const int units = batch * heads;
    const int grid = std::max(1, std::min(units, num_sms()));
    if (launch_pdl(attn_fwd_short_kernel, dim3(grid), dim3(SH_FWD_THREADS), SH_FWD_SMEM2, s, 1, tm, tmo, cu, batch,
                   heads, d, slopes, O, lse, nnz) != cudaSuccess)
      return MB_ERR_CUDA;
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  static const bool v1 = [] {  // MB_ATTN_LONG_FWD=v1: the round-1 one-query-tile kernel (A/B)
    const char* e = std::getenv("MB_ATTN_LONG_FWD");
    return e && e[0] == 'v' && e[1] == '1';
  }();
  if (!v1 && (size_t)batch * heads * ((max_seqlen + 2 * TILE - 1) / (2 * TILE)) <= (size_t)num_sms() * L2_UMAX) {
    static bool attr_2 = false;
    if (!attr_2) {
      if (cudaFuncSetAttribute(attn_fwd_long2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L2_SMEM) !=
          cudaSuccess)
        return MB_ERR_CUDA;
      attr_2 = true;
    }
    PairUnits P{cu, heads, (max_seqlen + 2 * TILE - 1) / (2 * TILE), 0};
    P.total = batch * heads * P.QP;
    const int grid = std::max(1, std::min(P.total, num_sms()));
    CUtensorMap tmo2;  // [32 rows x 32 columns] output blocks, 64-byte swizzle
    MB_REQUIRE(make_tmap_bf16_2d(&tmo2, O, H, nnz, H, 32, 32, 64), MB_ERR_CUDA);
    if (launch_pdl(attn_fwd_long2_kernel, dim3(grid), dim3(L2_THREADS), L2_SMEM, s, 1, tm, tmo2, P, d, slopes, O, lse,
                   nnz) != cudaSuccess)
      return MB_ERR_CUDA;
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  static bool attr_l = false;
  if (!attr_l) {
    if (cudaFuncSetAttribute(attn_fwd_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, LF_SMEM) !=
        cudaSuccess)
      return MB_ERR_CUDA;
    attr_l = true;
  }
  CUtensorMap tmo;
  MB_REQUIRE(make_tmap_bf16_2d(&tmo, O, H, nnz, H, 32, 32, 64), MB_ERR_CUDA);
  LongUnits U{cu, heads, (max_seqlen + TILE - 1) / TILE, 0};
  U.total = batch * heads * U.QT;
  const int grid = std::max(1, std::min(U.total, num_sms()));
  if (launch_pdl(attn_fwd_long_kernel, dim3(grid), dim3(LF_THREADS), LF_SMEM, s, 1, tm, tmo, U, d, slopes, O, lse,
                 nnz) != cudaSuccess)
    return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  return MB_OK;
}

// long path: dq_acc fp32 [nnz, H] (deterministic mode: one such slab per key tile) followed by D
// fp32 [heads, nnz].  Also sized for l <= 128: batches with more (sequence, head) units than the
// short backward's per-CTA unit lists hold run on the long kernel.
size_t attention_ws_bytes(int nnz, int heads, int d, int max_seqlen, bool det) {
  const size_t slabs = det ? (size_t)((std::max(max_seqlen, 1) + TILE - 1) / TILE) : 1;
  const size_t dq = (slabs * nnz * heads * d * sizeof(float) + 255) & ~size_t(255);
  return dq + (size_t)heads * nnz * sizeof(float);
}

mb_status attention_bwd(const bf16* qkv, const bf16* O, const bf16* dO, const float* lse, const int* cu, int batch,
                        int nnz, int max_seqlen, int heads, int d, const float* slopes, bf16* dqkv, float* dbias,
                        void* ws, size_t ws_bytes, cudaStream_t s, const Det* det) {
  if (nnz == 0 || batch == 0) return MB_OK;
  MB_REQUIRE(d == 32 || d == 64, MB_ERR_CONFIG);
  MB_REQUIRE(max_seqlen >= 1 && max_seqlen <= kMaxSeqlen, MB_ERR_SHAPE);
  const int H = heads * d;
  const bool dm = det && *det;
  const size_t need = attention_ws_bytes(nnz, heads, d, max_seqlen, dm);
  MB_REQUIRE(ws_bytes >= need && (need == 0 || ws), MB_ERR_WORKSPACE);
  if (dm && dbias) {  // deterministic mode: the kernels skip db_qkv; ordered column sums of dQ, dV afterwards
    MB_REQUIRE(det->part_floats >= colsum_det_floats(nnz, H), MB_ERR_WORKSPACE);
    mb_status st = attention_bwd(qkv, O, dO, lse, cu, batch, nnz, max_seqlen, heads, d, slopes, dqkv, nullptr, ws,
                                 ws_bytes, s, det);
    if (st != MB_OK) return st;
    if ((st = colsum_det(dqkv, 3 * H, nnz, H, dbias, det->part, s)) != MB_OK) return st;  // db_q (db_k = 0, R31)
    return colsum_det(dqkv + 2 * H, 3 * H, nnz, H, dbias + 2 * H, det->part, s);          // db_v
  }
  CUtensorMap tq, tdo;
  MB_REQUIRE(make_tmap_bf16_2d(&tq, qkv, 3 * H, nnz, 3 * H, DT, TILE), MB_ERR_CUDA);
  MB_REQUIRE(make_tmap_bf16_2d(&tdo, dO, H, nnz, H, DT, TILE), MB_ERR_CUDA);
  // short path: per-CTA unit lists hold BW_UMAX units (beyond: the long kernel, which takes any l)
  if (max_seqlen <= TILE && batch * heads <= std::max(1, std::min(batch * heads, num_sms())) * BW_UMAX) {
    CUtensorMap tdq;  // [32 rows x 32 columns] output blocks, 64-byte swizzle
    MB_REQUIRE(make_tmap_bf16_2d(&tdq, dqkv, 3 * H, nnz, 3 * H, 32, 32, 64), MB_ERR_CUDA);
    static bool attr_s = false;
    if (!attr_s) {
      if (cudaFuncSetAttribute(attn_bwd_short_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SH_BWD_SMEM) !=
          cudaSuccess)
        return MB_ERR_CUDA;
      attr_s = true;
    }
    const int units = batch * heads;
    const int grid = std::max(1, std::min(units, num_sms()));
    if (launch_pdl(attn_bwd_short_kernel, dim3(grid), dim3(SH_BWD_THREADS), SH_BWD_SMEM, s, 1, tq, tdo, tdq, cu,
                   batch, heads, d, slopes, O, dO, lse, dqkv, dbias, nnz) != cudaSuccess)
      return MB_ERR_CUDA;
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  static bool attr_l = false;
  if (!attr_l) {
    if (cudaFuncSetAttribute(attn_bwd_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, LB_SMEM) !=
        cudaSuccess)
      return MB_ERR_CUDA;
    attr_l = true;
  }
  const int QT = (max_seqlen + TILE - 1) / TILE;
  const size_t slabs = dm ? (size_t)QT : 1;  // deterministic mode: one fp32 dQ slab per key tile
  float* dq_acc = reinterpret_cast<float*>(ws);
  float* Dg = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                       ((slabs * nnz * H * sizeof(float) + 255) & ~size_t(255)));
  if (!dm && cudaMemsetAsync(dq_acc, 0, (size_t)nnz * H * sizeof(float), s) != cudaSuccess) return MB_ERR_CUDA;
  {
    MB_REQUIRE(H <= 1024, MB_ERR_CONFIG);  // the prep kernel's warp covers a row in at most 4 x 32 chunks
    attn_bwd_prep_kernel<<<(unsigned)std::max(1, std::min((nnz + 7) / 8, 8 * num_sms())), 256, 0, s>>>(O, dO, nnz,
                                                                                                       heads, d, Dg);
    MB_CHECK_LAUNCH();
  }
  CUtensorMap tdq, tdqa;  // [32 x 32] dK / dV bf16 blocks (64B swizzle); [32 x 32] fp32 dQ blocks (128B swizzle)
  MB_REQUIRE(make_tmap_bf16_2d(&tdq, dqkv, 3 * H, nnz, 3 * H, 32, 32, 64), MB_ERR_CUDA);
  MB_REQUIRE(make_tmap_f32_2d(&tdqa, dq_acc, H, slabs * nnz, H, 32, 32, 128), MB_ERR_CUDA);
  LongUnits U{cu, heads, QT, 0};
  U.total = batch * heads * U.QT;
  const int grid = std::max(1, std::min(U.total, num_sms()));
  if (launch_pdl(attn_bwd_long_kernel, dim3(grid), dim3(LB_THREADS), LB_SMEM, s, 1, tq, tdo, tdq, tdqa, U, d, slopes,
                 lse, Dg, dq_acc, dqkv, dbias, nnz, dm ? 1 : 0) != cudaSuccess)
    return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  if (dm) {
    dq_finish_det_kernel<<<(nnz + 7) / 8, dim3(H / 8, 8), 0, s>>>(dq_acc, cu, batch, nnz, H, dqkv);
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  {
    // one wave: two CTAs of (H/8) x 8 threads per SM, each covering an equal share of the rows
    const int slots = 2 * num_sms();
    const int rows_per = std::max(DQF_GROUPS, ((nnz + slots - 1) / slots + DQF_GROUPS - 1) / DQF_GROUPS * DQF_GROUPS);
    dq_finish_kernel<<<(nnz + rows_per - 1) / rows_per, dim3(H / 8, DQF_GROUPS), DQF_GROUPS * H * sizeof(float),
                       s>>>(dq_acc, nnz, H, rows_per, dqkv, dbias);
    MB_CHECK_LAUNCH();
  }
  return MB_OK;
}

}  // namespace mb

extern "C" {

mb_status mb_attention_forward(const mb_bf16* qkv, const int32_t* cu_seqlens, int32_t batch, int32_t nnz,
                               int32_t max_seqlen, int32_t heads, int32_t head_dim, const float* slopes, mb_bf16* O,
                               float* lse, mb_stream_t s) {
  if (!qkv || !cu_seqlens || !slopes || !O || !lse || batch < 0 || nnz < 0) return MB_ERR_INVALID_ARG;
  if (heads <= 0) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  return mb::attention_fwd(reinterpret_cast<const bf16*>(qkv), cu_seqlens, batch, nnz, max_seqlen, heads, head_dim,
                           slopes, reinterpret_cast<bf16*>(O), lse, reinterpret_cast<cudaStream_t>(s));
}

size_t mb_attention_workspace_bytes(int32_t nnz, int32_t heads, int32_t head_dim, int32_t max_seqlen) {
  return mb::attention_ws_bytes(nnz, heads, head_dim, max_seqlen, false);
}

mb_status mb_attention_backward(const mb_bf16* qkv, const mb_bf16* O, const mb_bf16* dO, const float* lse,
                                const int32_t* cu_seqlens, int32_t batch, int32_t nnz, int32_t max_seqlen,
                                int32_t heads, int32_t head_dim, const float* slopes, mb_bf16* dqkv, float* db_qkv,
                                void* ws, size_t ws_bytes, mb_stream_t s) {
  if (!qkv || !O || !dO || !lse || !cu_seqlens || !slopes || !dqkv || batch < 0 || nnz < 0)
    return MB_ERR_INVALID_ARG;
  if (heads <= 0) return MB_ERR_CONFIG;
  MB_REQUIRE_ARCH();
  return mb::attention_bwd(reinterpret_cast<const bf16*>(qkv), reinterpret_cast<const bf16*>(O),
                           reinterpret_cast<const bf16*>(dO), lse, cu_seqlens, batch, nnz, max_seqlen, heads,
                           head_dim, slopes, reinterpret_cast<bf16*>(dqkv), db_qkv, ws, ws_bytes,
                           reinterpret_cast<cudaStream_t>(s));
}

}  // extern "C"

#ifdef MB_TRACE_L2
extern "C" MB_API int mb_diag_l2_trace(long long* host) {  // diagnostic builds only
  if (cudaMemcpyFromSymbol(host, mb::l2_trace, sizeof(mb::l2_trace)) != cudaSuccess) return 1;
  return cudaMemcpyFromSymbol(host + 2 * 16 * 8, mb::l2_mtrace, sizeof(mb::l2_mtrace)) != cudaSuccess;
}
#endif
