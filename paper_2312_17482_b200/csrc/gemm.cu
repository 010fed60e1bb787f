// Persistent warp-specialised tcgen05 GEMM with fused epilogues.
//
//   warp 0      : TMA producer (one lane) — A/B tiles into a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      : MMA issuer (one lane)   — tcgen05.mma kind::f16, 128 x BN x 16 per instruction,
//                 accumulating in TMEM; double-buffered accumulator (2 x BN fp32 columns)
//   warp 2      : TMEM allocator
//   warps 4..11 : epilogue (two warps per TMEM lane quarter, one per half of the tile's columns) —
//                 tcgen05.ld 32 lanes x 32 columns, fused bias / residual / GeLU / GeGLU fwd+bwd /
//                 fp32 atomic accumulate; bf16 inputs and outputs move through a per-warp smem
//                 scratch so that every global access is coalesced (8 rows x 64 B per instruction)
//
// Operands may be K-major (the nn.Linear forward layout) or MN-major (the transposed operands of
// dX = dY W and dW = dY^T X); both are expressed with 128-byte-swizzled TMA boxes and the matching
// UMMA shared-memory descriptors, so no operand is ever transposed in memory.
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma.h"

namespace mb {
namespace {

constexpr int BM = 128, BK = 64;
constexpr int kSplitOverheadKb = 4;  // split-K cost model: one unit's fp32 flush ~ this many k-blocks
constexpr int NUM_EPI_WARPS = 8;                     // two warps per TMEM lane quarter
constexpr int NTHREADS = 128 + 32 * NUM_EPI_WARPS;  // warps 0-3: TMA, MMA, TMEM alloc, spare
// per-warp epilogue scratch: 32 rows x 32 bf16 (64 B), 16-byte unit u of row r stored at unit
// u ^ ((r >> 1) & 3): conflict-free both for row-wise access (lane = row, 8 rows per 128-byte phase)
// and for the coalescing pattern (8 lanes = 2 rows x 4 units per phase)
constexpr int SCR_ROW = 64;
constexpr int SCR_BYTES = 32 * SCR_ROW;
__device__ __forceinline__ uint32_t scr_at(uint32_t scr, int row, int unit) {
  return scr + row * SCR_ROW + ((unit ^ ((row >> 1) & 3)) << 4);
}

template <int BN, int STAGES, int NSCR, int CG = 1, int ACC = 2>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // a CTA pair splits B's N between its two CTAs
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int DATA = STAGE_BYTES * STAGES;
  static constexpr int SCR = NUM_EPI_WARPS * NSCR * SCR_BYTES;
  static constexpr int BIAS = NUM_EPI_WARPS * 256;  // per-warp staged bias slice of the current tile
  // no alignment slack: the dynamic shared window of these kernels starts 1024-byte aligned (no
  // static shared memory); the kernel traps if it ever does not
  static constexpr int SMEM = DATA + SCR + BIAS + 384;
  static constexpr int TMEM_NEED = ACC * BN;  // ACC accumulator stages of BN fp32 columns
  static constexpr int TMEM_COLS = TMEM_NEED <= 256 ? 256 : 512;
};

struct Sched {
  int num_m, num_n, splits, nkb, kb_per, total;
  __device__ __forceinline__ void decode(int u, int& m, int& n, int& kb0, int& kb1) const {
    const int tiles = num_m * num_n;
    const int s = u / tiles;
    const int t = u - s * tiles;
    m = t / num_n;
    n = t - m * num_n;
    kb0 = s * kb_per;
    kb1 = min(nkb, kb0 + kb_per);
  }
  // k-block range [d0, d1) of a unit whose A tiles also feed the bias gradient: the unit's range is
  // split evenly over the num_n column tiles of its m-block (db does not depend on n), so every
  // tile reads 1/num_n of its A tiles a second time instead of the n = 0 tiles reading all
  __device__ __forceinline__ void db_range(int n, int kb0, int kb1, int& d0, int& d1) const {
    const int len = (kb1 - kb0 + num_n - 1) / num_n;
    d0 = min(kb1, kb0 + n * len);
    d1 = min(kb1, d0 + len);
  }
};

__device__ __forceinline__ void load_bf16x32(const bf16* src, float* v, int ncols_valid) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (g * 8 < ncols_valid) {
      uint4 u = *reinterpret_cast<const uint4*>(src + g * 8);
      bf16x8_to_f32(u, v + g * 8);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[g * 8 + j] = 0.f;
    }
  }
}

// ---- warp-cooperative coalesced movement of a 32-row x 32-column bf16 chunk through a per-warp
// smem scratch: lane l covers rows (l>>2)+8i, 16-byte segment (l&3), so every global access
// instruction touches 8 full 64-byte row segments instead of 32 scattered half-sectors.
__device__ __forceinline__ void chunk_load(uint4 (&r)[4], const bf16* base, int64_t ld, int row0, int M, int col,
                                           int N, int lane) {
  const int c = col + (lane & 3) * 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = row0 + (lane >> 2) + 8 * i;
    if (row < M && c < N) r[i] = *reinterpret_cast<const uint4*>(base + (int64_t)row * ld + c);
    else r[i] = make_uint4(0, 0, 0, 0);
  }
}
// explicit shared-window accesses (the scratch lives behind a 1024-aligned dynamic-smem pointer, so
// plain C++ dereferences would compile to generic LD.E/ST.E)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ void sts128(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void chunk_to_scr(uint32_t scr, const uint4 (&r)[4], int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) sts128(scr_at(scr, (lane >> 2) + 8 * i, lane & 3), r[i]);
}
__device__ __forceinline__ void scr_row_read(uint32_t scr, int lane, float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) bf16x8_to_f32(lds128(scr_at(scr, lane, j)), v + 8 * j);
}
__device__ __forceinline__ void scr_row_write(uint32_t scr, int lane, const float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) sts128(scr_at(scr, lane, j), f32_to_bf16x8(v + 8 * j));
}
__device__ __forceinline__ void scr_to_global(uint32_t scr, bf16* base, int64_t ld, int row0, int M, int col, int N,
                                              int lane) {
  const int c = col + (lane & 3) * 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = (lane >> 2) + 8 * i;
    const int row = row0 + rr;
    const uint4 v = lds128(scr_at(scr, rr, lane & 3));
    if (row < M && c < N) *reinterpret_cast<uint4*>(base + (int64_t)row * ld + c) = v;
  }
}
// row-wise values of this lane -> scratch -> coalesced global store
__device__ __forceinline__ void emit_chunk(uint32_t scr, const float* v, bf16* base, int64_t ld, int row0, int M,
                                           int col, int N, int lane) {
  scr_row_write(scr, lane, v);
  __syncwarp();
  scr_to_global(scr, base, ld, row0, M, col, N, lane);
  __syncwarp();
}

__device__ __forceinline__ void stg256(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
               "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void load_bias32_smem(uint32_t sb, float* v) {
#pragma unroll
  for (int g = 0; g < 4; ++g) bf16x8_to_f32(lds128(sb + g * 16), v + g * 8);
}

// per-warp transpose-reduce: lane l ends with the sum over the warp's 32 rows of column l of v[32]
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

// CG = 2: the CTA pair of a 2-CTA cluster computes a 256 x BN tile with tcgen05.mma.cta_group::2
// (M = 256): each CTA loads its 128 rows of A and its half of B's N (halving per-SM operand
// ingest per FLOP), the pair leader (cluster rank 0) issues the MMAs, and each CTA's TMEM holds the
// accumulator rows of its own half.
// ACC = 2 double-buffers the TMEM accumulator (epilogue of tile i overlaps the MMAs of tile i+1);
// ACC = 1 is used by the weight-gradient GEMMs, whose tiles run hundreds of k-blocks per (cheap)
// epilogue, to make room in TMEM for the bias-gradient accumulator.
template <int BN, int STAGES, int A_MN, int B_MN, int PAIRED, int NSCR, int CG, int ACC, int CE>
__global__ void __launch_bounds__(NTHREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX, int M, int N,
                Sched sc, Epi ep) {
  using C = Cfg<BN, STAGES, NSCR, CG, ACC>;
  static_assert(ACC == 2 || A_MN == 1, "the fused bias gradient reads MN-major A tiles");
  extern __shared__ uint8_t smem_raw[];
  if (sm100::smem_u32(smem_raw) & 1023) __trap();  // Cfg::SMEM reserves no alignment slack
  uint8_t* smem = smem_raw;
  uint8_t* scr_base = smem + C::DATA;
  uint8_t* bias_base = smem + C::DATA + C::SCR;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DATA + C::SCR + C::BIAS);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* mdone = tempty + 2;  // [STAGES] (ACC == 1) the MMAs have consumed the stage
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mdone + STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = CG == 2 ? (int)sm100::cluster_ctarank() : 0;
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;  // this CTA's cluster and the cluster count

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    if (PAIRED || ep.tma_store) sm100::tma_prefetch(&tmC);
    if (PAIRED) sm100::tma_prefetch(&tmX);
    // ACC == 1 (weight gradients with a fused bias gradient): the MMA's commit goes to mdone and the
    // epilogue warps, after reading the stage's A tile for db, release it to the producer (empty)
    for (int i = 0; i < STAGES; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], ACC == 1 ? NUM_EPI_WARPS : 1);
      if (ACC == 1) sm100::mbar_init(&mdone[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], NUM_EPI_WARPS * CG);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) {
    if (CG == 2) sm100::tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    else sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  sm100::tc_fence_before();
  if (CG == 2) sm100::cluster_sync();
  else __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // everything above touched only shared memory, TMEM and kernel parameters
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < sc.total; u += ncl) {
        int mb, nb, kb0, kb1;
        sc.decode(u, mb, nb, kb0, kb1);
        const int m_cta = (mb * CG + rank) * BM;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], CG * C::STAGE_BYTES);
          const int k0 = kb * BK;
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if (CG == 2) sm100::tma_load_2d_pair(dst, m, &full[stage], c0, c1);
            else sm100::tma_load_2d(dst, m, &full[stage], c0, c1);
          };
          if (!A_MN) {
            load(sa, &tmA, k0, m_cta);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) load(sa + i * 8192, &tmA, m_cta + i * 64, k0);
          }
          if (PAIRED) {
            if (CG == 2) {
              load(sb, &tmB, k0, rank * ep.I + nb * 128);  // leader: W1 rows (a), peer: V rows (g)
            } else {
              load(sb, &tmB, k0, nb * 128);
              load(sb + 128 * 128, &tmB, k0, ep.I + nb * 128);
            }
          } else if (!B_MN) {
            load(sb, &tmB, k0, nb * BN + rank * (BN / CG));
          } else {
#pragma unroll
            for (int i = 0; i < BN / CG / 64; ++i) load(sb + i * 8192, &tmB, nb * BN + rank * (BN / CG) + i * 64, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // the whole warp runs the issue loop; one elected lane issues
      constexpr uint32_t idesc = sm100::idesc_bf16(BM * CG, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cid; u < sc.total; u += ncl) {
        int mb, nb, kb0, kb1;
        sc.decode(u, mb, nb, kb0, kb1);
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? sm100::desc_mnmajor_sw128(sa + k * 2048, 8192) : sm100::desc_kmajor_sw128(sa + k * 32);
            const uint64_t bd = B_MN ? sm100::desc_mnmajor_sw128(sb + k * 2048, 8192) : sm100::desc_kmajor_sw128(sb + k * 32);
            if (CG == 2) sm100::mma_bf16_ss_pair_w(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            else sm100::mma_bf16_ss_w(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          uint64_t* rel = ACC == 1 ? &mdone[stage] : &empty[stage];
          if (CG == 2) sm100::mma_commit_pair_w(rel);
          else sm100::mma_commit_w(rel);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2) sm100::mma_commit_pair_w(&tfull[acc]);
        else sm100::mma_commit_w(&tfull[acc]);
        if (++acc == ACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;     // TMEM lane quarter this warp may access
    const int grp = ew >> 2;    // which half of the tile's columns
    const uint32_t scrA = sm100::smem_u32(scr_base) + ew * NSCR * SCR_BYTES;
    const uint32_t scrB = scrA + (NSCR > 1 ? SCR_BYTES : 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int rstage = 0;  // ACC == 1: position in the operand ring, in step with the MMA warp
    uint32_t rphase = 0;
    for (int u = cid; u < sc.total; u += ncl) {
      int mb, nb, kb0, kb1;
      sc.decode(u, mb, nb, kb0, kb1);
      if (ACC == 1) {
        // bias gradient of a weight-gradient GEMM, db[m] = sum_k A[m, k], on the CUDA cores from the
        // A tiles the MMAs have just consumed (MN-major: two 128B-swizzled boxes of 64 m x 64 k per
        // stage).  Thread t sums 16-byte chunk (t & 15) = 8 consecutive m over k-rows (t >> 4) + 16j.
        int dkb0 = 0, dkb1 = 0;
        if (ep.dbias) sc.db_range(nb, kb0, kb1, dkb0, dkb1);
        const int t = threadIdx.x - 128, ch = t & 15, r0 = t >> 4;
        float dbs[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) dbs[e] = 0.f;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&mdone[rstage], rphase);
          if (kb >= dkb0 && kb < dkb1) {
            const uint32_t sa = sm100::smem_u32(smem + rstage * C::STAGE_BYTES) + (ch >> 3) * 8192;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r = r0 + 16 * j;
              float f[8];
              bf16x8_to_f32(lds128(sa + r * 128 + (((ch & 7) ^ (r & 7)) << 4)), f);
#pragma unroll
              for (int e = 0; e < 8; ++e) dbs[e] += f[e];
            }
          }
          sm100::fence_proxy_async_smem();  // generic reads of the stage before the producer's next TMA write
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&empty[rstage]);
          if (++rstage == STAGES) {
            rstage = 0;
            rphase ^= 1;
          }
        }
        if (ep.dbias && ep.dpart) {
          // deterministic mode: the 8 warps' partials (same 128 rows, different k-rows) meet in shared
          // memory and warp 4 writes one partial per (split, column tile), summed in order later
#pragma unroll
          for (int e = 0; e < 8; ++e) dbs[e] += __shfl_xor_sync(0xffffffffu, dbs[e], 16);
          if (lane < 16) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(scrA + (lane * 8 + e) * 4), "f"(dbs[e]) : "memory");
          }
          asm volatile("bar.sync 1, %0;" ::"r"(32 * NUM_EPI_WARPS) : "memory");
          if (ew == 0 && lane < 16) {
            const uint32_t s0 = sm100::smem_u32(scr_base);
            float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int w = 0; w < NUM_EPI_WARPS; ++w) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                float x;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(s0 + w * NSCR * SCR_BYTES + (lane * 8 + e) * 4));
                acc8[e] += x;
              }
            }
            const int m0 = (mb * CG + rank) * BM + lane * 8;
            float* dp = ep.dpart + (int64_t)(kb0 / sc.kb_per * sc.num_n + nb) * M;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (m0 + e < M) dp[m0 + e] = acc8[e];
          }
          asm volatile("bar.sync 1, %0;" ::"r"(32 * NUM_EPI_WARPS) : "memory");
        } else if (ep.dbias && dkb0 < dkb1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) dbs[e] += __shfl_xor_sync(0xffffffffu, dbs[e], 16);
          const int m0 = (mb * CG + rank) * BM + ch * 8;
          if (lane < 16) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (m0 + e < M) atomicAdd(ep.dbias + m0 + e, dbs[e]);
          }
        }
      }
      const int row0 = (mb * CG + rank) * BM + q * 32;
      const int row = row0 + lane;
      const bool row_ok = row < M;
      // stage this tile's bias slice in smem (async, overlapped with the MMA of the tile): L1 is
      // nearly all carved out for the operand ring, so per-chunk bias reads would go to L2
      const uint32_t sbias = sm100::smem_u32(bias_base) + ew * 256;
      if (ep.bias && lane < 16) {
        if (PAIRED) {
          const int c = lane >> 3, t = (lane >> 2) & 1, seg = lane & 3;
          cp_async16(sbias + (c * 2 + t) * 64 + seg * 16, ep.bias + t * ep.I + nb * 128 + grp * 64 + c * 32 + seg * 8);
        } else {
          const int c = lane >> 2, seg = lane & 3;
          const int col = nb * BN + grp * (BN / 2) + c * 32 + seg * 8;
          if (c < BN / 64 && col < N) {
            if (col + 8 <= N) {
              cp_async16(sbias + c * 64 + seg * 16, ep.bias + col);
            } else {  // ragged last vector (N % 8 != 0): never read past the bias array
              for (int e = 0; e < 8; ++e) {
                const bf16 bv = col + e < N ? ep.bias[col + e] : __float2bfloat16(0.f);
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(sbias + c * 64 + seg * 16 + 2 * e),
                             "h"(*reinterpret_cast<const unsigned short*>(&bv)));
              }
            }
          }
        }
      }
      uint4 pa[4], pg[4];  // first input chunk (residual / Gd), prefetched before the accumulator is ready
      if (!PAIRED) {
        const int cbase0 = nb * BN + grp * (BN / 2);
        if (ep.mode == E_GEGLU_BWD) {
          chunk_load(pa, ep.U, ep.ldu, row0, M, cbase0, N, lane);
          chunk_load(pg, ep.U + ep.I, ep.ldu, row0, M, cbase0, N, lane);
        } else if (ep.mode == E_BF16 && ep.res) {
          chunk_load(pa, ep.res, ep.ldr, row0, M, cbase0, N, lane);
        }
      }
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      if (ep.bias) cp_async_wait_all();
      __syncwarp();
      const uint32_t tb = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      float v[32];
      if (PAIRED) {
        // paired tile: TMEM cols [0,128) = a (W1 half), [128,256) = g (V half); this warp group
        // owns a-columns [grp*64, grp*64+64) of the 128 output columns nb*128..
        float g[32];
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          const int crel = grp * 64 + c * 32;
          const int col = nb * 128 + crel;
          sm100::tmem_ld32(tb + crel, v);
          sm100::tmem_ld32(tb + 128 + crel, g);
          float ba[32], bg[32];
          load_bias32_smem(sbias + (c * 2 + 0) * 64, ba);
          load_bias32_smem(sbias + (c * 2 + 1) * 64, bg);
          sm100::tmem_ld_wait();
          if (c == 1) {  // last TMEM read of the tile: the MMAs of the tile after next may start
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (CG == 2) sm100::mbar_arrive_leader(&tempty[acc]);
              else sm100::mbar_arrive(&tempty[acc]);
            }
          }
#pragma unroll
          // output Z = GeLU(a) * g; saved for backward Gd = [g * GeLU'(a) | GeLU(a)] (the two factors
          // of dU = [dZ g GeLU'(a) | dZ GeLU(a)], so the backward epilogue needs no transcendental).
          // Two columns at a time on the paired fp32 pipe (FFMA2/FMUL2): this epilogue is ALU-bound.
          float z[32];
#ifndef MB_DIAG_GEGLU
#define MB_DIAG_GEGLU 0
#endif
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            if (MB_DIAG_GEGLU == 1 || MB_DIAG_GEGLU == 4) {  // diagnostic builds only: no GeLU math
              z[j] = v[j] * g[j]; z[j + 1] = v[j + 1] * g[j + 1];
              continue;
            }
            const float2 x = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(ba[j], ba[j + 1]));
            const float2 gg = __fadd2_rn(make_float2(g[j], g[j + 1]), make_float2(bg[j], bg[j + 1]));
            float2 cdf, pdf;
            norm_cdf_pdf2(x, cdf, pdf);
            const float2 ge = __fmul2_rn(x, cdf);
            const float2 zz = __fmul2_rn(ge, gg);
            const float2 gd = __fmul2_rn(gg, __ffma2_rn(x, pdf, cdf));
            z[j] = zz.x; z[j + 1] = zz.y;
            v[j] = gd.x; v[j + 1] = gd.y;
            g[j] = ge.x; g[j + 1] = ge.y;
          }
          if (MB_DIAG_GEGLU >= 3) {  // diagnostic builds only: keep the values alive, store nothing
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) s += z[j] + v[j] + g[j];
            if (s == 1234.5f) reinterpret_cast<bf16*>(ep.C)[row] = __float2bfloat16(s);
            continue;
          }
          // the three [32 x 32] outputs leave by TMA stores from the warp's three 64B-swizzled
          // scratch blocks (the scr_at layout is the TMA 64-byte swizzle); a block is rewritten only
          // after the store issued from it three emits earlier has read it
          auto emit_tma = [&](int slot, const float* val, const CUtensorMap* tm, int c0) {
            const uint32_t buf = scrA + slot * SCR_BYTES;
            if (lane == 0) sm100::bulk_wait_read<NSCR - 1>();
            __syncwarp();
            scr_row_write(buf, lane, val);
            sm100::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              sm100::tma_store_2d(tm, buf, c0, row0);
              sm100::bulk_commit();
            }
          };
          if (MB_DIAG_GEGLU != 2) {
            emit_tma(0, v, &tmX, col);
            emit_tma(1, g, &tmX, ep.I + col);
          }
          emit_tma(2, z, &tmC, col);
        }
      } else {
        constexpr int HALF = BN / 2;
        const int cbase = nb * BN + grp * HALF;
        // fused cross-entropy state (E_LSE / E_DZ)
        const bool ce = CE && (ep.mode == E_LSE || ep.mode == E_DZ);  // compiled only into CE kernels
        int lab = -1;
        float lse_r = 0.f, run_m = -INFINITY, run_s = 0.f, zl = 0.f;
        bool has_lab = false;
        if (ce && row_ok) {
          lab = ep.labels[row];
          if (ep.mode == E_DZ) lse_r = ep.lse[row];
        }
        constexpr float L2E = 1.4426950408889634f;
        // deterministic split-K: this tile's splits add into C one after another, in split order
        int* semp = nullptr;
        if (ep.mode == E_F32_ACC && ep.sem && sc.splits > 1) {
          const int tiles = sc.num_m * sc.num_n;
          semp = ep.sem + (u % tiles) * CG + rank;
          const int need = NUM_EPI_WARPS * (u / tiles);
          if (lane == 0) {
            // bounded wait: a turnstile that never opens (a scheduling bug) traps instead of hanging
            for (long long spin = 0; ld_acquire_s32(semp) < need; ++spin) {
              __nanosleep(64);
              if (spin > (1ll << 27)) __trap();
            }
          }
          __syncwarp();
        }
#pragma unroll 1
        for (int c = 0; c < HALF / 32; ++c) {
          const int crel = grp * HALF + c * 32;
          const int col = cbase + c * 32;
          if (col >= N) break;  // warp-uniform
          sm100::tmem_ld32(tb + crel, v);
          const int nv = min(32, N - col);
          if (CE && ce) {
            float b[32];
            load_bias32_smem(sbias + c * 64, b);
            sm100::tmem_ld_wait();
            if (ep.mode == E_LSE) {
              // online (max, sum exp) over this chunk; exponentials in the log2 domain, two columns
              // per instruction on the paired fp32 pipe
              float mx = -INFINITY;
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 z = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(b[j], b[j + 1]));
                v[j] = col + j < N ? z.x : -INFINITY;
                v[j + 1] = col + j + 1 < N ? z.y : -INFINITY;
                mx = fmaxf(mx, fmaxf(v[j], v[j + 1]));
              }
              if (lab >= col && lab < col + 32) {  // warp-divergent but rare: this row's label column
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col + j == lab) zl = v[j];
                has_lab = true;
              }
              const float nm = fmaxf(run_m, mx);
              const float nml = -nm * L2E;
              float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 t = __ffma2_rn(make_float2(v[j], v[j + 1]), make_float2(L2E, L2E), make_float2(nml, nml));
                acc2 = __fadd2_rn(acc2, make_float2(ex2_approx(t.x), ex2_approx(t.y)));
              }
              run_s = run_s * ex2_approx((run_m - nm) * L2E) + (acc2.x + acc2.y);
              run_m = nm;
            } else {
              const float nl = -lse_r * L2E;
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 z = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(b[j], b[j + 1]));
                const float2 t = __ffma2_rn(z, make_float2(L2E, L2E), make_float2(nl, nl));
                float2 pz = make_float2(ex2_approx(t.x), ex2_approx(t.y));
                if (col + j == lab) pz.x -= 1.f;
                if (col + j + 1 == lab) pz.y -= 1.f;
                pz = __fmul2_rn(pz, make_float2(ep.inv_norm, ep.inv_norm));
                v[j] = pz.x;
                v[j + 1] = pz.y;
              }
              if (ep.tma_store) {  // dz block by TMA store from the warp's scratch (see E_BF16)
                if (lane == 0) sm100::bulk_wait_read<0>();
                __syncwarp();
                scr_row_write(scrA, lane, v);
                sm100::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  sm100::tma_store_2d(&tmC, scrA, col, row0);
                  sm100::bulk_commit();
                }
              } else {
                emit_chunk(scrA, v, reinterpret_cast<bf16*>(ep.C), ep.ldc, row0, M, col, N, lane);
              }
            }
          } else if (ep.mode == E_F32_ACC) {
            sm100::tmem_ld_wait();
            if (row_ok) {
              float* dst = reinterpret_cast<float*>(ep.C) + (int64_t)row * ep.ldc + col;
              if (semp) {  // sole writer of these elements while this split holds the turnstile
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  if (j < nv) {
                    float4 o = __ldcg(reinterpret_cast<const float4*>(dst + j));
                    o.x += v[j], o.y += v[j + 1], o.z += v[j + 2], o.w += v[j + 3];
                    __stcg(reinterpret_cast<float4*>(dst + j), o);
                  }
              } else {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  if (j < nv) red_add_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
              }
            }
          } else if (ep.mode == E_F32) {
            float b[32];
            if (ep.bias) load_bias32_smem(sbias + c * 64, b);
            sm100::tmem_ld_wait();
            if (ep.bias) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += b[j];
            }
            if (row_ok) {
              float* dst = reinterpret_cast<float*>(ep.C) + (int64_t)row * ep.ldc + col;
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                if (j < nv) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            }
          } else if (ep.mode == E_GEGLU_BWD) {
            // v = dZ; saved Gd row holds g GeLU'(a) at [col..], GeLU(a) at [I+col..]  ->  dU = dZ * Gd
            chunk_to_scr(scrA, pa, lane);
            chunk_to_scr(scrB, pg, lane);
            __syncwarp();
            if (c + 1 < HALF / 32) {
              chunk_load(pa, ep.U, ep.ldu, row0, M, col + 32, N, lane);
              chunk_load(pg, ep.U + ep.I, ep.ldu, row0, M, col + 32, N, lane);
            }
            sm100::tmem_ld_wait();
            // 16 columns at a time keeps the live register set small (a, g, dZ)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float a[16], g[16];
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                bf16x8_to_f32(lds128(scr_at(scrA, lane, 2 * h + j)), a + 8 * j);
                bf16x8_to_f32(lds128(scr_at(scrB, lane, 2 * h + j)), g + 8 * j);
              }
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float dz = v[16 * h + j];
                a[j] = dz * a[j];  // dZ * g * GeLU'(a)
                g[j] = dz * g[j];  // dZ * GeLU(a)
              }
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                sts128(scr_at(scrA, lane, 2 * h + j), f32_to_bf16x8(a + 8 * j));
                sts128(scr_at(scrB, lane, 2 * h + j), f32_to_bf16x8(g + 8 * j));
              }
            }
            __syncwarp();
            bf16* D = reinterpret_cast<bf16*>(ep.C);
            scr_to_global(scrA, D, ep.ldc, row0, M, col, N, lane);
            scr_to_global(scrB, D + ep.I, ep.ldc, row0, M, col, N, lane);
            if (ep.dbias) {
              // db_1v = column sums of dU (the rounded values that were stored), fused here:
              // transpose-reduce over the warp's 32 rows, one atomic per column per warp
              float t[32];
              scr_row_read(scrA, lane, t);
#pragma unroll
              for (int j = 0; j < 32; ++j) t[j] = row_ok ? t[j] : 0.f;
              const float ca = warp_colsum32(t, lane);
              scr_row_read(scrB, lane, t);
#pragma unroll
              for (int j = 0; j < 32; ++j) t[j] = row_ok ? t[j] : 0.f;
              const float cg = warp_colsum32(t, lane);
              if (col + lane < N) {
                atomicAdd(ep.dbias + col + lane, ca);
                atomicAdd(ep.dbias + ep.I + col + lane, cg);
              }
            }
            __syncwarp();
          } else {  // E_BF16 / E_GELU_AUX
            float b[32];
            if (ep.bias) load_bias32_smem(sbias + c * 64, b);
            if (ep.res) {
              chunk_to_scr(scrA, pa, lane);
              __syncwarp();
              if (c + 1 < HALF / 32) chunk_load(pa, ep.res, ep.ldr, row0, M, col + 32, N, lane);
            }
            sm100::tmem_ld_wait();
            if (ep.bias) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += b[j];
            }
            if (CE == 2 && row_ok) {  // F2 dropout of the projection output, before the residual
#pragma unroll
              for (int g8 = 0; g8 < 4; ++g8) dropout_apply8(ep.drop, (uint32_t)row, (uint32_t)(col + 8 * g8), v + 8 * g8);
            }
            if (ep.res) {
              float r[32];
              scr_row_read(scrA, lane, r);
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += r[j];
            }
            if (ep.mode == E_GELU_AUX) {
              emit_chunk(scrA, v, ep.aux, ep.ldaux, row0, M, col, N, lane);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
            }
            if (ep.tma_store && ep.mode == E_BF16) {
              // the output [32 x 32] block leaves by a TMA store from the warp's last scratch block
              // (64B swizzle = the scr_at layout; the first one stages the residual when NSCR == 2),
              // once the previous chunk's store has read it
              if (lane == 0) sm100::bulk_wait_read<0>();
              __syncwarp();
              scr_row_write(scrB, lane, v);
              sm100::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                sm100::tma_store_2d(&tmC, scrB, col, row0);
                sm100::bulk_commit();
              }
            } else {
              emit_chunk(scrA, v, reinterpret_cast<bf16*>(ep.C), ep.ldc, row0, M, col, N, lane);
            }
          }
        }
        if (CE && ep.mode == E_LSE && row_ok) {
          ep.part[(int64_t)row * ep.npart + nb * 2 + grp] = make_float2(run_m, run_s);
          if (has_lab) ep.zlab[row] = zl;
        }
        if (semp) {  // pass the turnstile on; the last split's last warp resets it for the next GEMM
          __syncwarp();
          if (lane == 0) {
            __threadfence();
            if (atomicAdd(semp, 1) == NUM_EPI_WARPS * sc.splits - 1) atomicExch(semp, 0);
          }
        }
      }
      if (!PAIRED) {  // (the paired epilogue released its accumulator after its last TMEM read)
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) sm100::mbar_arrive_leader(&tempty[acc]);
          else sm100::mbar_arrive(&tempty[acc]);
        }
      }
      if (++acc == ACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if ((PAIRED || ep.tma_store) && lane == 0) sm100::bulk_wait0();  // the TMA stores have left shared memory
  }
  sm100::tc_fence_before();
  if (CG == 2) sm100::cluster_sync();
  else __syncthreads();
  sm100::tc_fence_after();
  if (warp == 2) {
    if (CG == 2) sm100::tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    else sm100::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}


// ------------------------------------------------------------------------------------------------
// GeGLU backward (A8 bwd, epilogue E4) as a dedicated kernel with asynchronous epilogue I/O:
//   dZ = dF W2 (tcgen05, never stored);  dU = dZ * Gd,  Gd = [g GeLU'(a) | GeLU(a)] saved by the
//   forward.  (db_1v = column sums of dU comes from the dW1v GEMM's tensor-core row sums.)
// A CTA pair computes 256 rows x 256 columns of dZ (cta_group::2, each CTA 128 rows x all 256
// columns in TMEM, double-buffered).  The wide tile halves the MMA operand ingest per FLOP of the
// former 128-column tile, which matters because this kernel is bounded by the SM's shared-memory
// bandwidth: operands + Gd in (TMA) + Gd read + dU write + dU out (TMA) all cross it.  The epilogue
// walks the tile in four 64-column quarters; a dedicated producer warp streams each quarter's Gd
// slice ([128 x 64] of each half, 32 KB) into a 4-slot ring ahead of use, the 8 epilogue warps
// multiply in place (swizzled layout) and one thread TMA-stores the quarter, releasing its slot
// once the store has read it.  Warps: 0 operand TMA, 1 MMA, 2 TMEM alloc, 3 Gd TMA, 4-11 epilogue.
// ------------------------------------------------------------------------------------------------
#ifndef MB_GB_STAGES
#define MB_GB_STAGES 4
#endif
#ifndef MB_GB_NSLOT
#define MB_GB_NSLOT 3
#endif
constexpr int GB_BN = 256, GB_STAGES = MB_GB_STAGES, GB_NSLOT = MB_GB_NSLOT;
constexpr int GB_STAGE_BYTES = BM * BK * 2 + (GB_BN / 2) * BK * 2;  // own 128 A rows + half of B (32 KB)
constexpr int GB_SLOT_BYTES = 2 * BM * 64 * 2;                      // a and g boxes [128 x 64] bf16 (32 KB)
constexpr int GB_SMEM = GB_STAGES * GB_STAGE_BYTES + GB_NSLOT * GB_SLOT_BYTES + 1024 + 256;

// Default (DIRECT_STORE = false): dU is written in place over the Gd slot, and the two warps of each
// TMEM lane quarter meet on a 64-thread named barrier after which one lane TMA-stores their [32 x 64]
// rows of both boxes (coalesced, 128B swizzle = the in-place layout); a slot goes back to the loader
// once its four quarter leaders' stores have read it.  DIRECT_STORE (MB_GEGLU_BWD_STORE=direct):
// dU leaves the registers by row-per-thread 32-byte stores and each Gd slot is released as soon as the
// 8 warps have read it (fewer shared-memory passes, faster in isolation, 0.5 % slower in the step)
template <bool DIRECT_STORE>
__global__ void __launch_bounds__(NTHREADS, 1)
    geglu_bwd_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmGd, const __grid_constant__ CUtensorMap tmDU, int M, int I,
                     Sched sc, bf16* __restrict__ dU) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* slots = smem + GB_STAGES * GB_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + GB_NSLOT * GB_SLOT_BYTES);
  uint64_t* empty = full + GB_STAGES;
  uint64_t* tfull = empty + GB_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* gfull = tempty + 2;        // [GB_NSLOT] Gd quarter landed (own CTA)
  uint64_t* gempty = gfull + GB_NSLOT;  // [GB_NSLOT] slot's dU store has read it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gempty + GB_NSLOT);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = (int)sm100::cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    sm100::tma_prefetch(&tmGd);
    sm100::tma_prefetch(&tmDU);
    for (int i = 0; i < GB_STAGES; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], 2 * NUM_EPI_WARPS);
    }
    for (int i = 0; i < GB_NSLOT; ++i) {
      sm100::mbar_init(&gfull[i], 1);
      sm100::mbar_init(&gempty[i], DIRECT_STORE ? NUM_EPI_WARPS : 4);  // TMA: the 4 quarter leaders
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair(tmem_slot, 2 * GB_BN);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // everything above touched only shared memory, TMEM and kernel parameters
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // operands: own 128 rows of dF, own half (128 columns) of W2's tile
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < sc.total; u += ncl) {
        int mb, nb, kb0, kb1;
        sc.decode(u, mb, nb, kb0, kb1);
        const int m_cta = (mb * 2 + rank) * BM;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * GB_STAGE_BYTES;
          uint8_t* sb = sa + BM * BK * 2;
          if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], 2 * GB_STAGE_BYTES);
          const int k0 = kb * BK;
          sm100::tma_load_2d_pair(sa, &tmA, &full[stage], k0, m_cta);
#pragma unroll
          for (int i = 0; i < GB_BN / 2 / 64; ++i)
            sm100::tma_load_2d_pair(sb + i * 8192, &tmB, &full[stage], nb * GB_BN + rank * (GB_BN / 2) + i * 64, k0);
          if (++stage == GB_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // Gd quarters of this CTA's rows, GB_NSLOT ahead
      int qi = 0;
      for (int u = cid; u < sc.total; u += ncl) {
        int mb, nb, kb0, kb1;
        sc.decode(u, mb, nb, kb0, kb1);
        const int m_cta = (mb * 2 + rank) * BM;
        for (int qq = 0; qq < GB_BN / 64; ++qq, ++qi) {
          const int sl = qi % GB_NSLOT;
          sm100::mbar_wait(&gempty[sl], ((qi / GB_NSLOT) & 1) ^ 1);
          uint8_t* slot = slots + sl * GB_SLOT_BYTES;
          sm100::mbar_arrive_expect_tx(&gfull[sl], GB_SLOT_BYTES);
          sm100::tma_load_2d(slot, &tmGd, &gfull[sl], nb * GB_BN + qq * 64, m_cta);
          sm100::tma_load_2d(slot + BM * 128, &tmGd, &gfull[sl], I + nb * GB_BN + qq * 64, m_cta);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // the whole warp runs the issue loop; one elected lane issues
      constexpr uint32_t idesc = sm100::idesc_bf16(2 * BM, GB_BN, 0, 1);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cid; u < sc.total; u += ncl) {
        int mb, nb, kb0, kb1;
        sc.decode(u, mb, nb, kb0, kb1);
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * GB_BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + stage * GB_STAGE_BYTES);
          const uint32_t sb = sa + BM * BK * 2;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            sm100::mma_bf16_ss_pair_w(d_tmem, sm100::desc_kmajor_sw128(sa + k * 32),
                                    sm100::desc_mnmajor_sw128(sb + k * 2048, 8192), idesc,
                                    (kb > kb0 || k > 0) ? 1u : 0u);
          sm100::mma_commit_pair_w(&empty[stage]);
          if (++stage == GB_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        sm100::mma_commit_pair_w(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;   // TMEM lane quarter = rows [32q, 32q+32) of this CTA's half
    const int grp = ew >> 2;  // 32-column half of each 64-column quarter
    const int gtid = threadIdx.x - 128;  // 0..255
    const int r = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int qi = 0;
    for (int u = cid; u < sc.total; u += ncl) {
      int mb, nb, kb0, kb1;
      sc.decode(u, mb, nb, kb0, kb1);
      const int row0 = (mb * 2 + rank) * BM;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      for (int qq = 0; qq < GB_BN / 64; ++qq, ++qi) {
        const int sl = qi % GB_NSLOT;
        const uint32_t box_a = sm100::smem_u32(slots + sl * GB_SLOT_BYTES), box_g = box_a + BM * 128;
        float v[32];
        sm100::tmem_ld32(tmem_base + acc * GB_BN + ((uint32_t)(q * 32) << 16) + qq * 64 + grp * 32, v);
        sm100::mbar_wait(&gfull[sl], (qi / GB_NSLOT) & 1);
        sm100::tmem_ld_wait();
        if (qq == GB_BN / 64 - 1) {  // accumulator fully read: the MMA may reuse it
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive_leader(&tempty[acc]);
        }
        // dU = dZ * Gd in place: row r, 16-byte chunks grp*4 .. grp*4+3 of the 64-column box (swizzled)
        uint4 A[4], G[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = grp * 4 + jj;
          const uint32_t off = r * 128 + ((j ^ (r & 7)) << 4);
          A[jj] = lds128(box_a + off);
          G[jj] = lds128(box_g + off);
        }
        if (DIRECT_STORE) {
          uint4 oa[4], og[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            float ga[8], gg[8];
            bf16x8_to_f32(A[jj], ga);
            bf16x8_to_f32(G[jj], gg);
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 dz = make_float2(v[8 * jj + e], v[8 * jj + e + 1]);
              const float2 pa = __fmul2_rn(dz, make_float2(ga[e], ga[e + 1]));
              const float2 pg = __fmul2_rn(dz, make_float2(gg[e], gg[e + 1]));
              ga[e] = pa.x, ga[e + 1] = pa.y, gg[e] = pg.x, gg[e + 1] = pg.y;
            }
            oa[jj] = f32_to_bf16x8(ga);
            og[jj] = f32_to_bf16x8(gg);
          }
          // the slot's values have been consumed (the products depend on every loaded register):
          // order the generic-proxy reads before the producer's next TMA write, then hand it back
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive(&gempty[sl]);
          if (row0 + r < M) {
            bf16* da = dU + (size_t)(row0 + r) * (2 * I) + nb * GB_BN + qq * 64 + grp * 32;
            stg256(da, oa[0], oa[1]);
            stg256(da + 16, oa[2], oa[3]);
            stg256(da + I, og[0], og[1]);
            stg256(da + I + 16, og[2], og[3]);
          }
          continue;
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = grp * 4 + jj;
          const uint32_t off = r * 128 + ((j ^ (r & 7)) << 4);
          float ga[8], gg[8];
          bf16x8_to_f32(A[jj], ga);
          bf16x8_to_f32(G[jj], gg);
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float2 dz = make_float2(v[8 * jj + e], v[8 * jj + e + 1]);
            const float2 pa = __fmul2_rn(dz, make_float2(ga[e], ga[e + 1]));
            const float2 pg = __fmul2_rn(dz, make_float2(gg[e], gg[e + 1]));
            ga[e] = pa.x, ga[e + 1] = pa.y, gg[e] = pg.x, gg[e + 1] = pg.y;
          }
          sts128(box_a + off, f32_to_bf16x8(ga));
          sts128(box_g + off, f32_to_bf16x8(gg));
        }
        // the two warps of this lane quarter (32 rows x 64 columns of the box) meet, and one lane
        // TMA-stores their rows of both boxes ([32 x 64], 128B swizzle = the in-place layout)
        sm100::fence_proxy_async_smem();
        sm100::named_bar(2 + q, 64);
        if (grp == 0 && lane == 0) {
          sm100::tma_store_2d(&tmDU, box_a + q * 4096, nb * GB_BN + qq * 64, row0 + q * 32);
          sm100::tma_store_2d(&tmDU, box_g + q * 4096, I + nb * GB_BN + qq * 64, row0 + q * 32);
          sm100::bulk_commit();
          if (qi > 0) {  // the previous quarter's stores have read their slot: hand it back
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            sm100::mbar_arrive(&gempty[(qi - 1) % GB_NSLOT]);
          }
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (!DIRECT_STORE && grp == 0 && lane == 0) {
      sm100::bulk_wait_read0();
      if (qi > 0) sm100::mbar_arrive(&gempty[(qi - 1) % GB_NSLOT]);
      sm100::bulk_wait0();
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  if (warp == 2) sm100::tmem_dealloc_pair(tmem_base, 2 * GB_BN);
}


template <int BN, int STAGES, int A_MN, int B_MN, int PAIRED, int NSCR, int CG = 2, int ACC = 2, int CE = 0>
mb_status launch(const GemmArgs& g, const CUtensorMap& ta, const CUtensorMap& tb, const Sched& sc, cudaStream_t s,
                 const CUtensorMap* tc = nullptr, const CUtensorMap* tx = nullptr) {
  using C = Cfg<BN, STAGES, NSCR, CG, ACC>;
  auto k = gemm_kernel<BN, STAGES, A_MN, B_MN, PAIRED, NSCR, CG, ACC, CE>;
  static bool attr_set = false;  // benign race: idempotent
  if (!attr_set) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess)
      return MB_ERR_CUDA;
    attr_set = true;
  }
  const int clusters = std::max(1, std::min(sc.total, num_sms() / CG));
  if (launch_pdl(k, dim3(clusters * CG), dim3(NTHREADS), C::SMEM, s, CG, ta, tb, tc ? *tc : ta, tx ? *tx : ta, g.M,
                 g.N, sc, g.ep) != cudaSuccess)
    return MB_ERR_CUDA;
  MB_CHECK_LAUNCH();
  return MB_OK;
}

template <int BN, int STAGES, int NSCR>
mb_status dispatch_majors(const GemmArgs& g, const CUtensorMap& ta, const CUtensorMap& tb, const Sched& sc,
                          cudaStream_t s) {
  if (!g.a_t && !g.b_t) return launch<BN, STAGES, 0, 0, 0, NSCR>(g, ta, tb, sc, s);
  if (!g.a_t && g.b_t) return launch<BN, STAGES, 0, 1, 0, NSCR>(g, ta, tb, sc, s);
  if (g.a_t && g.b_t) return launch<BN, STAGES, 1, 1, 0, NSCR>(g, ta, tb, sc, s);
  return launch<BN, STAGES, 1, 0, 0, NSCR>(g, ta, tb, sc, s);
}

}  // namespace

mb_status gemm(const GemmArgs& g, cudaStream_t s) {
  MB_REQUIRE(g.A && g.B && g.ep.C, MB_ERR_INVALID_ARG);
  MB_REQUIRE(g.M >= 0 && g.N >= 0 && g.K >= 0, MB_ERR_INVALID_ARG);
  if (g.M == 0 || g.N == 0) return MB_OK;
  MB_REQUIRE(g.K > 0, MB_ERR_INVALID_ARG);
  // N % 8 != 0 only for the decoder's fused-CE GEMMs (any vocabulary, F3): their bf16 output rows
  // are padded (ldc >= N rounded up to 8), so the last 16-byte vector of a row stays inside it
  const bool ce_any = g.ep.mode == E_LSE || g.ep.mode == E_DZ;
  MB_REQUIRE(g.lda % 8 == 0 && g.ldb % 8 == 0, MB_ERR_CONFIG);
  MB_REQUIRE(g.N % 8 == 0 || (ce_any && g.ep.ldc >= ((g.N + 7) & ~7)), MB_ERR_CONFIG);
  const bool paired = g.ep.mode == E_GEGLU_FWD;
  if (paired) MB_REQUIRE(g.ep.I % 128 == 0 && g.N == 2 * g.ep.I && !g.a_t && !g.b_t, MB_ERR_CONFIG);
  if (g.ep.mode == E_GEGLU_BWD) MB_REQUIRE(g.N == g.ep.I, MB_ERR_CONFIG);

  // BN: 256 for wide outputs, 128 when N is small (tiny configs); GeGLU fwd is always a 256-wide
  // paired tile (128 columns of W1 + the matching 128 of V), GeGLU bwd a 256-wide tile.
  const bool geglu_bwd = g.ep.mode == E_GEGLU_BWD;
  const bool ce_mode = g.ep.mode == E_LSE || g.ep.mode == E_DZ;  // partial-statistics layout assumes 256
  const bool drop_mode = g.ep.mode == E_BF16 && g.ep.drop.thr;  // F2 variant exists for BN = 256 only
  const int BN = (paired || ce_mode || drop_mode || geglu_bwd) ? 256 : (g.N <= 128 ? 128 : 256);
  // CG = 2 (generic kernel): pair tiles of 256 rows; each CTA loads 128 rows of A and BN/2 of B's N.
  constexpr int CGV = 2;
  CUtensorMap ta, tb;
  bool ok;
  if (!g.a_t) ok = make_tmap_bf16_2d(&ta, g.A, g.K, g.M, g.lda, BK, BM);
  else ok = make_tmap_bf16_2d(&ta, g.A, g.M, g.K, g.lda, 64, BK);
  MB_REQUIRE(ok, MB_ERR_CUDA);
  if (paired) ok = make_tmap_bf16_2d(&tb, g.B, g.K, g.N, g.ldb, BK, 128);
  else if (!g.b_t) ok = make_tmap_bf16_2d(&tb, g.B, g.K, g.N, g.ldb, BK, geglu_bwd ? BN : BN / CGV);
  else ok = make_tmap_bf16_2d(&tb, g.B, g.N, g.K, g.ldb, 64, BK);
  MB_REQUIRE(ok, MB_ERR_CUDA);

  Sched sc;
  sc.num_m = (g.M + (geglu_bwd ? BM : BM * CGV) - 1) / (geglu_bwd ? BM : BM * CGV);
  sc.num_n = paired ? g.ep.I / 128 : (g.N + BN - 1) / BN;
  sc.nkb = (g.K + BK - 1) / BK;
  int splits = 1;
  if (g.ep.mode == E_F32_ACC) {
    // split-K for the weight gradients (few output tiles, K = tokens): pick the split count S that
    // minimises waves(S) x (k-blocks per unit + a per-unit epilogue overhead): a 2.07-wave launch
    // idles 1/3 of the machine in its last wave, while every extra split adds an fp32-atomic tile
    // flush; >= 8 k-blocks per split. Partial sums meet in fp32 atomics (the += contract).
    const int tiles = sc.num_m * sc.num_n;
    const int C = std::max(1, num_sms() / CGV);
    double best = 1e30;
    for (int S = 1; S <= std::max(1, std::min(64, sc.nkb / 8)); ++S) {
      const int kbp = (sc.nkb + S - 1) / S;
      const int units = tiles * ((sc.nkb + kbp - 1) / kbp);
      const double cost = (double)((units + C - 1) / C) * (kbp + kSplitOverheadKb);
      if (cost < best * 0.98) { best = cost; splits = S; }
    }
    if (const char* e = getenv("MB_SPLITK")) splits = std::max(1, std::min(atoi(e), sc.nkb));  // tuning only
  }
  sc.kb_per = (sc.nkb + splits - 1) / splits;
  sc.splits = (sc.nkb + sc.kb_per - 1) / sc.kb_per;
  sc.total = sc.num_m * sc.num_n * sc.splits;
  GemmArgs gd = g;  // deterministic mode: turnstile counters for split-K, partial slab for the fused db
  const bool det = g.det && *g.det && g.ep.mode == E_F32_ACC;
  if (det) {
    if (sc.splits > 1) {
      MB_REQUIRE(g.det->sem && g.det->sem_count >= sc.num_m * sc.num_n * CGV, MB_ERR_WORKSPACE);
      gd.ep.sem = g.det->sem;
    }
    if (g.ep.dbias) {
      MB_REQUIRE(g.det->part_floats >= (size_t)sc.splits * sc.num_n * g.M, MB_ERR_WORKSPACE);
      gd.ep.dpart = g.det->part;
    }
  }

  if (paired) {  // outputs Z [M, I] and Gd [M, 2I] leave by TMA stores of [32 x 32] 64B-swizzled blocks
    CUtensorMap tz, tgd;
    MB_REQUIRE(make_tmap_bf16_2d(&tz, g.ep.C, g.ep.I, g.M, g.ep.ldc, 32, 32, 64), MB_ERR_CUDA);
    MB_REQUIRE(make_tmap_bf16_2d(&tgd, g.ep.aux, 2 * g.ep.I, g.M, g.ep.ldaux, 32, 32, 64), MB_ERR_CUDA);
    return launch<256, 5, 0, 0, 1, 3>(g, ta, tb, sc, s, &tz, &tgd);
  }
  if (geglu_bwd) {
    if (g.a_t || !g.b_t || g.ep.I % GB_BN || g.ep.ldu != 2 * g.ep.I || g.ep.ldc != 2 * g.ep.I) return MB_ERR_CONFIG;
    CUtensorMap tg, tdu;
    MB_REQUIRE(make_tmap_bf16_2d(&tg, g.ep.U, 2 * g.ep.I, g.M, g.ep.ldu, 64, BM), MB_ERR_CUDA);
    MB_REQUIRE(make_tmap_bf16_2d(&tdu, g.ep.C, 2 * g.ep.I, g.M, g.ep.ldc, 64, 32), MB_ERR_CUDA);  // per lane quarter
    // default: dU written in place into the Gd slot and TMA-stored per lane quarter (C2 step +0.5 %
    // against row-per-thread 32-byte stores in a same-box A/B); MB_GEGLU_BWD_STORE=direct: the stores
    static const bool direct = [] {
      const char* e = std::getenv("MB_GEGLU_BWD_STORE");
      return e && e[0] == 'd';
    }();
    auto kern = direct ? geglu_bwd_kernel<true> : geglu_bwd_kernel<false>;
    static bool attr_gb = false;
    if (!attr_gb) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GB_SMEM) != cudaSuccess)
        return MB_ERR_CUDA;
      attr_gb = true;
    }
    Sched sg = sc;  // pair tiles of 256 rows
    sg.num_m = (g.M + 2 * BM - 1) / (2 * BM);
    sg.total = sg.num_m * sg.num_n * sg.splits;
    const int clusters = std::max(1, std::min(sg.total, num_sms() / 2));
    if (launch_pdl(kern, dim3(2 * clusters), dim3(NTHREADS), GB_SMEM, s, 2, ta, tb, tg, tdu, g.M, g.ep.I, sg,
                   reinterpret_cast<bf16*>(g.ep.C)) != cudaSuccess)
      return MB_ERR_CUDA;
    MB_CHECK_LAUNCH();
    return MB_OK;
  }
  if (g.ep.mode == E_F32_ACC && g.a_t && g.b_t && g.ep.dbias) {  // wgrad + fused db: 1 accumulator
    const mb_status st = BN == 256 ? launch<256, 6, 1, 1, 0, 1, 2, 1>(gd, ta, tb, sc, s)
                                   : launch<128, 8, 1, 1, 0, 1, 2, 1>(gd, ta, tb, sc, s);
    if (st != MB_OK || !gd.ep.dpart) return st;
    return ordered_sum(gd.ep.dpart, sc.splits * sc.num_n, g.M, g.M, g.ep.dbias, s);
  }
  MB_REQUIRE(g.ep.dbias == nullptr, MB_ERR_INVALID_ARG);
  if (g.ep.mode == E_LSE || g.ep.mode == E_DZ) {  // decoder GEMM with fused softmax-cross-entropy
    MB_REQUIRE(!g.a_t && !g.b_t && g.ep.labels && g.ep.bias && BN == 256, MB_ERR_CONFIG);
    MB_REQUIRE(g.ep.mode == E_DZ ? g.ep.lse != nullptr : (g.ep.part && g.ep.zlab), MB_ERR_INVALID_ARG);
    if (g.ep.mode == E_DZ && g.ep.ldc % 8 == 0 && (reinterpret_cast<uintptr_t>(g.ep.C) & 15) == 0) {
      CUtensorMap tc;  // dz [M, N] (row stride ldc): [32 x 32] blocks, 64-byte swizzle; columns >= N clipped
      MB_REQUIRE(make_tmap_bf16_2d(&tc, g.ep.C, g.N, g.M, g.ep.ldc, 32, 32, 64), MB_ERR_CUDA);
      GemmArgs gt = g;
      gt.ep.tma_store = 1;
      return launch<256, 6, 0, 0, 0, 1, 2, 2, 1>(gt, ta, tb, sc, s, &tc);
    }
    return launch<256, 6, 0, 0, 0, 1, 2, 2, 1>(g, ta, tb, sc, s);
  }
  if (g.ep.mode == E_BF16 && g.ep.drop.thr) {  // F2: bias -> dropout -> residual (forward projections)
    MB_REQUIRE(!g.a_t && !g.b_t && BN == 256, MB_ERR_CONFIG);
    return launch<256, 6, 0, 0, 0, 1, 2, 2, 2>(g, ta, tb, sc, s);
  }
  if (BN == 256 && g.ep.mode == E_BF16 && !g.a_t && g.ep.ldc % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(g.ep.C) & 15) == 0) {
    // forward / dX GEMMs: output by TMA stores; with a residual two scratch blocks per epilogue warp
    // and without one a single block, both with the 6-stage ring
    CUtensorMap tc;
    MB_REQUIRE(make_tmap_bf16_2d(&tc, g.ep.C, g.N, g.M, g.ep.ldc, 32, 32, 64), MB_ERR_CUDA);
    GemmArgs gt = gd;
    gt.ep.tma_store = 1;
    if (g.ep.res) return g.b_t ? launch<256, 6, 0, 1, 0, 2>(gt, ta, tb, sc, s, &tc)
                                : launch<256, 6, 0, 0, 0, 2>(gt, ta, tb, sc, s, &tc);
    return g.b_t ? launch<256, 6, 0, 1, 0, 1>(gt, ta, tb, sc, s, &tc) : launch<256, 6, 0, 0, 0, 1>(gt, ta, tb, sc, s, &tc);
  }
  if (BN == 256) return dispatch_majors<256, 6, 1>(gd, ta, tb, sc, s);
  return dispatch_majors<128, 8, 1>(gd, ta, tb, sc, s);
}

size_t gemm_det_floats(int M, int N, int K) {
  // fused-db partial slab bound: splits <= 64 (the split-K search), column tiles of 128
  (void)K;
  return (size_t)64 * (size_t)((N + 127) / 128) * (size_t)M;
}
int gemm_det_sems(int M, int N) { return 2 * ((M + 255) / 256) * ((N + 127) / 128); }

}  // namespace mb

extern "C" mb_status mb_gemm(int32_t M, int32_t N, int32_t K, const mb_bf16* A, int64_t lda, int32_t a_t,
                             const mb_bf16* B, int64_t ldb, int32_t b_t, void* C, int64_t ldc, int32_t epilogue,
                             const mb_bf16* bias, const mb_bf16* residual, int64_t ldr, mb_bf16* aux, int64_t ldaux,
                             mb_stream_t s) {
  MB_REQUIRE(A && B && C, MB_ERR_INVALID_ARG);
  MB_REQUIRE_ARCH();
  mb::GemmArgs g;
  g.M = M, g.N = N, g.K = K;
  g.A = reinterpret_cast<const bf16*>(A), g.lda = lda, g.a_t = a_t != 0;
  g.B = reinterpret_cast<const bf16*>(B), g.ldb = ldb, g.b_t = b_t != 0;
  switch (epilogue) {
    case MB_EPI_BF16: g.ep.mode = mb::E_BF16; break;
    case MB_EPI_F32_ACC: g.ep.mode = mb::E_F32_ACC; break;
    case MB_EPI_F32: g.ep.mode = mb::E_F32; break;
    case MB_EPI_GELU_AUX: g.ep.mode = mb::E_GELU_AUX; MB_REQUIRE(aux, MB_ERR_INVALID_ARG); break;
    default: return MB_ERR_INVALID_ARG;
  }
  g.ep.C = C, g.ep.ldc = ldc;
  g.ep.bias = reinterpret_cast<const bf16*>(bias);
  g.ep.res = reinterpret_cast<const bf16*>(residual), g.ep.ldr = ldr;
  g.ep.aux = reinterpret_cast<bf16*>(aux), g.ep.ldaux = ldaux;
  return mb::gemm(g, reinterpret_cast<cudaStream_t>(s));
}

extern "C" mb_status mb_gemm_wgrad(int32_t M, int32_t N, int32_t K, const mb_bf16* dY, int64_t lda, const mb_bf16* X,
                                   int64_t ldb, float* dW, int64_t ldc, float* db, mb_stream_t s) {
  MB_REQUIRE(dY && X && dW, MB_ERR_INVALID_ARG);
  MB_REQUIRE_ARCH();
  mb::GemmArgs g;
  g.M = M, g.N = N, g.K = K;
  g.A = reinterpret_cast<const bf16*>(dY), g.lda = lda, g.a_t = true;
  g.B = reinterpret_cast<const bf16*>(X), g.ldb = ldb, g.b_t = true;
  g.ep.mode = mb::E_F32_ACC, g.ep.C = dW, g.ep.ldc = ldc, g.ep.dbias = db;
  return mb::gemm(g, reinterpret_cast<cudaStream_t>(s));
}

extern "C" mb_status mb_geglu_forward(const mb_bf16* X, int32_t n, int32_t H, int32_t I, const mb_bf16* w_1v,
                                      const mb_bf16* b_1v, mb_bf16* Gd, mb_bf16* Z, mb_stream_t s) {
  MB_REQUIRE(X && w_1v && b_1v && Gd && Z, MB_ERR_INVALID_ARG);
  MB_REQUIRE_ARCH();
  mb::GemmArgs g;
  g.M = n, g.N = 2 * I, g.K = H;
  g.A = reinterpret_cast<const bf16*>(X), g.lda = H;
  g.B = reinterpret_cast<const bf16*>(w_1v), g.ldb = H;
  g.ep.mode = mb::E_GEGLU_FWD;
  g.ep.C = Z, g.ep.ldc = I;
  g.ep.bias = reinterpret_cast<const bf16*>(b_1v);
  g.ep.aux = reinterpret_cast<bf16*>(Gd), g.ep.ldaux = 2 * I;
  g.ep.I = I;
  return mb::gemm(g, reinterpret_cast<cudaStream_t>(s));
}

extern "C" mb_status mb_geglu_backward(const mb_bf16* dF, int32_t n, int32_t H, int32_t I, const mb_bf16* w_2,
                                       const mb_bf16* Gd, mb_bf16* dU, mb_stream_t s) {
  MB_REQUIRE(dF && w_2 && Gd && dU, MB_ERR_INVALID_ARG);
  MB_REQUIRE_ARCH();
  mb::GemmArgs g;
  g.M = n, g.N = I, g.K = H;
  g.A = reinterpret_cast<const bf16*>(dF), g.lda = H;
  g.B = reinterpret_cast<const bf16*>(w_2), g.ldb = I, g.b_t = true;  // W2 [H, I] = [K, N]
  g.ep.mode = mb::E_GEGLU_BWD;
  g.ep.C = dU, g.ep.ldc = 2 * I;
  g.ep.U = reinterpret_cast<const bf16*>(Gd), g.ep.ldu = 2 * I;
  g.ep.I = I;
  return mb::gemm(g, reinterpret_cast<cudaStream_t>(s));
}
