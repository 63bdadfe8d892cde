// tc.cu — BF16 mode on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Type I ("level kernel"): one launch per batching task V_t (Alg. 1).
//   D[unit j, vertex n] = sum_k A[j, k] * B[n, k]  with A = weights (K-major, TMA),
//   B = the task's contiguous rows of a position-ordered arena (K-major, TMA) — swap-AB,
//   so the tensor-core M side (128) is gate units and the small, ragged task size M_t is
//   the N side (tile NT = 64).  Accumulators live in TMEM; the epilogue stages them in
//   shared memory, transposed so one thread owns 4 consecutive units of one vertex, and
//   runs the whole cell (cells.cuh: gates, activations, child-sum, scatter, push) with
//   16-byte accesses — §3.5's kernel fusion done by hand across the GEMM.
//   U h~ = sum_k U h_k is accumulated in TMEM (reading Z11), so no h~ operand is formed.
//   Two variants:
//   * CL = 1 (monolithic): one CTA = 128 units x all gates (the large x-projection / dX);
//   * CL = 4 (gate split): a 4-CTA cluster splits a 128-unit block by gate (forward
//     i/o/u/f, backward and dX the K columns of each gate), so each CTA streams 1/4 of the
//     weights; accumulators are exchanged through distributed shared memory and rank r
//     finishes task columns [16r, 16r+16) (the per-level tasks).
//   Warp roles: w0 TMA producer, w1 TMEM allocator + single-thread MMA issuer,
//   w2..w9 per-vertex metadata, then epilogue.
// Type II ("lazy GEMM"): the deferred parameter gradients batched over ALL vertices
//   (lazy batching): out[m, n] = sum_p A[p, m] B[p, n] with both operands
//   MN-major straight from the position-ordered arenas, split-K across CTAs.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "cells.cuh"
#include "gemm.h"
#include "lazy.h"
#include "rows.h"
#include "persist.h"
#include "ptx.cuh"
#include "tc.h"

namespace cavs {

constexpr int NT = 64;                     // task-row tile (MMA N) of type I
constexpr int BK = 64;                     // k-block: one 128-byte swizzle atom of bf16
constexpr int A_TILE = 128 * BK * 2;       // 16 KB
constexpr int B_TILE = NT * BK * 2;        // 8 KB
constexpr int kThreads = 320;              // 10 warps
constexpr int kSmemBudget = 196 * 1024;    // pipeline stages (+ static metadata <= 227 KB)
constexpr int kCluster = 4;                // gate-split cluster: one rank per gate group
constexpr int kClMax = 16;                 // K-sliced gate split: kCluster x ksl ranks (ksl in {1, 2, 4})

struct Bundle {
  int map_a;                 // which A tensor map (0/1)
  int nA; int a_row[4];      // A row offsets (added to the CTA's unit base m0)
  int a_col0;                // A column (k) base
  int nB; int b_col[4];      // B column bases in the arena
  int nk;                    // k-blocks
  int nmma; int mma_a[8], mma_b[8], mma_acc[8];
};
struct RankPlan { int nb; Bundle b[3]; int nacc; int stages; int stage_bytes; int offB; };
// CL = 1: rank 0 only; CL = kCluster: one plan per rank.  comb[e][r] = accumulator of rank r
// summed into epilogue slot e (-1: none).
// npair = 6 in the FP32 split mode (bf16x3 operands): every bundle's k-loop runs
// once per plane pair (s, t) with s + t <= 2, A plane s at A row + s a_prow[map], B plane t at task
// row + t b_prow (plane-major arenas); npair = 1: plain bf16.
// kpb > 0 (grouped stages, r02): the maps are 4-D {64 k, rows, k-block, plane} and a stage holds kpb
// consecutive k-blocks of every A and B tile in all planes, ONE TMA box per tile (one SM's boxes are
// serviced one after another, ~0.3 us each: fewer, larger boxes; tools/tma_tile).  kpb = 0: the 2-D
// per-k-block maps (legacy path).
struct PlanT { RankPlan r[kClMax]; int comb[8][kClMax]; int bar_off; int npair; int a_prow[2]; int b_prow; int kpb; };
__device__ __constant__ const int kPairS[6] = {0, 0, 1, 0, 1, 2};
__device__ __constant__ const int kPairT[6] = {0, 1, 0, 2, 1, 0};

struct SegT2 { int a_col; int b_col; int k_lo, k_hi; int skip_no_x; };
// planes = 3 (split mode): a stage holds the three planes of the A and B tiles (plane q of an arena starts
// q * vp rows after plane 0), the six plane-pair products are issued from it, corrections into a
// second accumulator
struct PlanII { int nseg; SegT2 s[4]; int M, Ncols, ldo; int split; size_t split_stride; int stages; int accum;
                int planes; int vp; };

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~(uintptr_t)1023);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}

// ------------------------------------------------------------------------------------
// Type-I kernel.  CL = 1 (monolithic) or kCluster (gate split).
template <int E, int NACC, int CL, class OpT>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_level(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
           const __grid_constant__ CUtensorMap mB, Dev D, PlanT P, int row_lo, int row_hi, int units) {
  constexpr int COLS = NT / CL;                        // task columns finished by this CTA
  constexpr bool PM = is_s3<OpT>::value;               // split mode: plane-major stages (P.npair == 6)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const uint32_t rank = CL > 1 ? cluster_rank() : 0;
  const RankPlan& R = P.r[rank];
  const int S = R.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bar_off);
  uint64_t* empty = full + 6;
  uint64_t* done = empty + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* xs = reinterpret_cast<float*>(smem);          // [nacc][NT][128] after the mainloop
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (blockIdx.x / CL) * 128;
  const int p0 = row_lo + blockIdx.y * NT;
  const int c_own = (int)rank * COLS;                  // first task column finished here
  __shared__ VMeta s_meta[COLS];
  __shared__ unsigned long long s_tr[3];
  if (D.trace && threadIdx.x == 0) s_tr[0] = gtime();

  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ || E == EPI_DX) {
    bool act = false;                                  // uniform across a cluster (same task tile)
    if (threadIdx.x < NT) { const int p = p0 + threadIdx.x; act = p < row_hi && row_active<E>(D, p, D.xrow_pos[p]); }
    if (!__syncthreads_or(act)) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch(&mA0); ptx::tma_prefetch(&mA1); ptx::tma_prefetch(&mB);
      ptx::griddep_wait();
      if (D.trace) s_tr[2] = gtime();
      ptx::griddep_launch();                           // PDL: let the next task's CTAs start their prologue
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
      uint32_t written = 0;                            // accumulators already initialised
      int step = 0;
      constexpr int PS[6] = {0, 0, 1, 0, 1, 2}, PT[6] = {0, 1, 0, 2, 1, 0};
      if (P.kpb > 0) {
        // grouped stages: tile (plane q, k-block j) of operand i at base_i + (q kpb + j) * TILE
        const int kpb = P.kpb, np = P.npair > 1 ? 3 : 1;
        for (int bi = 0; bi < R.nb; ++bi) {
          const Bundle& b = R.b[bi];
          for (int g0 = 0; g0 < b.nk; g0 += kpb, ++step) {
            const int s = step % S;
            ptx::mbar_wait(&full[s], (step / S) & 1);
            ptx::tc_fence_after();
            const uint32_t st = ptx::smem_u32(smem + s * R.stage_bytes);
            const int kn = min(kpb, b.nk - g0);
            for (int jj = 0; jj < kn; ++jj)
              for (int m = 0; m < b.nmma; ++m)
                for (int pr = 0; pr < P.npair; ++pr) {
                  const uint32_t a = st + ((b.mma_a[m] * np + PS[pr]) * kpb + jj) * A_TILE;
                  const uint32_t bb = st + R.offB + ((b.mma_b[m] * np + PT[pr]) * kpb + jj) * B_TILE;
                  const int acc = b.mma_acc[m] + (pr > 0 ? R.nacc : 0);
                  const uint32_t d = tmem + acc * NT;
#pragma unroll
                  for (int kk = 0; kk < BK / 16; ++kk)
                    ptx::mma_bf16(d, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(bb + kk * 32, 16, 1024),
                                  idesc, ((written >> acc) & 1u) | (kk > 0 ? 1u : 0u));
                  written |= 1u << acc;
                }
            ptx::mma_commit(&empty[s]);
          }
        }
      } else if constexpr (PM) {
        // split mode: a stage holds the three planes of every A and B tile of the k-block, the six
        // plane-pair products a_s b_t (s + t <= 2) are issued from it (each plane loaded once)
        for (int bi = 0; bi < R.nb; ++bi) {
          const Bundle& b = R.b[bi];
          for (int kb = 0; kb < b.nk; ++kb, ++step) {
            const int s = step % S;
            ptx::mbar_wait(&full[s], (step / S) & 1);
            ptx::tc_fence_after();
            const uint32_t st = ptx::smem_u32(smem + s * R.stage_bytes);
            for (int m = 0; m < b.nmma; ++m) {
#pragma unroll
              for (int pr = 0; pr < 6; ++pr) {
                const uint32_t a = st + (PS[pr] * b.nA + b.mma_a[m]) * A_TILE;
                const uint32_t bb = st + R.offB + (PT[pr] * b.nB + b.mma_b[m]) * B_TILE;
                const int acc = b.mma_acc[m] + (pr > 0 ? R.nacc : 0);
                const uint32_t d = tmem + acc * NT;
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  ptx::mma_bf16(d, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(bb + kk * 32, 16, 1024),
                                idesc, ((written >> acc) & 1u) | (kk > 0 ? 1u : 0u));
                written |= 1u << acc;
              }
            }
            ptx::mma_commit(&empty[s]);
          }
        }
      } else
      for (int bi = 0; bi < R.nb; ++bi)
      for (int pr = 0; pr < P.npair; ++pr) {
        const Bundle& b = R.b[bi];
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&full[s], ph);
          ptx::tc_fence_after();
          const uint32_t st = ptx::smem_u32(smem + s * R.stage_bytes);
          for (int m = 0; m < b.nmma; ++m) {
            const uint32_t a = st + b.mma_a[m] * A_TILE;
            const uint32_t bb = st + R.offB + b.mma_b[m] * B_TILE;
            // split mode: the five correction products (pairs 1..5, ~2^-8 of the main one) accumulate
            // separately (acc + nacc): the tensor core's fp32 accumulation then adds them into a small
            // sum, and the main chain a0 b0 keeps plain bf16 MMA's number of accumulation steps
            const int acc = b.mma_acc[m] + (pr > 0 ? R.nacc : 0);
            const uint32_t d = tmem + acc * NT;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              ptx::mma_bf16(d, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(bb + kk * 32, 16, 1024),
                            idesc, ((written >> acc) & 1u) | (kk > 0 ? 1u : 0u));
            written |= 1u << acc;
          }
          ptx::mma_commit(&empty[s]);
        }
      }
      ptx::mma_commit(done);
    }
    __syncwarp();
  } else {
    if (lane == 0) {
      // ---- TMA issue, one warp per pipeline stage (a single issuing thread serialises its
      // boxes): stage s = warp - 2 owns steps s, s+S, ... so each stage's barrier phases
      // advance strictly in order.  Weight (A) tiles do not depend on the previous task, so
      // under PDL they stream in before griddepcontrol.wait; the task's rows (B) after it.
      const int w = warp - 2;
      bool waited = false;
      int step = 0;
      if (P.kpb > 0) {
        // grouped stages: ONE 4-D box {64, rows, kpb, planes} per A / B tile of the stage
        const int kpb = P.kpb, np = P.npair > 1 ? 3 : 1;
        for (int bi = 0; bi < R.nb; ++bi) {
          const Bundle& b = R.b[bi];
          const CUtensorMap* ma = b.map_a ? &mA1 : &mA0;
          for (int g0 = 0; g0 < b.nk; g0 += kpb, ++step) {
            if (step % S != w) continue;
            const int s = step % S;
            uint8_t* st = smem + s * R.stage_bytes;
            if (step >= S) ptx::mbar_wait(&empty[s], ((step / S) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(&full[s], np * kpb * (b.nA * A_TILE + b.nB * B_TILE));
            for (int i = 0; i < b.nA; ++i)
              ptx::tma_load_4d(st + i * np * kpb * A_TILE, ma, 0, b.a_row[i] + m0, b.a_col0 / BK + g0, 0, &full[s]);
            if (!waited) { ptx::griddep_wait(); waited = true; }
            for (int i = 0; i < b.nB; ++i)
              ptx::tma_load_4d(st + R.offB + i * np * kpb * B_TILE, &mB, 0, p0, b.b_col[i] / BK + g0, 0, &full[s]);
          }
        }
      } else if constexpr (PM) {
        for (int bi = 0; bi < R.nb; ++bi) {
          const Bundle& b = R.b[bi];
          const CUtensorMap* ma = b.map_a ? &mA1 : &mA0;
          for (int kb = 0; kb < b.nk; ++kb, ++step) {
            if (step % S != w) continue;
            const int s = step % S;
            uint8_t* st = smem + s * R.stage_bytes;
            if (step >= S) ptx::mbar_wait(&empty[s], ((step / S) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(&full[s], 3 * (b.nA * A_TILE + b.nB * B_TILE));
            for (int q = 0; q < 3; ++q)
              for (int i = 0; i < b.nA; ++i)
                ptx::tma_load_2d(st + (q * b.nA + i) * A_TILE, ma, b.a_col0 + kb * BK,
                                 b.a_row[i] + m0 + q * P.a_prow[b.map_a], &full[s]);
            if (!waited) { ptx::griddep_wait(); waited = true; }
            for (int q = 0; q < 3; ++q)
              for (int i = 0; i < b.nB; ++i)
                ptx::tma_load_2d(st + R.offB + (q * b.nB + i) * B_TILE, &mB, b.b_col[i] + kb * BK,
                                 p0 + q * P.b_prow, &full[s]);
          }
        }
      } else
      for (int bi = 0; bi < R.nb; ++bi)
      for (int pr = 0; pr < P.npair; ++pr) {
        const Bundle& b = R.b[bi];
        const CUtensorMap* ma = b.map_a ? &mA1 : &mA0;
        const int arow = m0 + kPairS[pr] * P.a_prow[b.map_a], brow = p0 + kPairT[pr] * P.b_prow;
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          if (step % S != w) continue;
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          uint8_t* st = smem + s * R.stage_bytes;
          if (step >= S) ptx::mbar_wait(&empty[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], b.nA * A_TILE + b.nB * B_TILE);
          for (int i = 0; i < b.nA; ++i)
            ptx::tma_load_2d(st + i * A_TILE, ma, b.a_col0 + kb * BK, b.a_row[i] + arow, &full[s]);
          if (!waited) { ptx::griddep_wait(); waited = true; }
          for (int i = 0; i < b.nB; ++i)
            ptx::tma_load_2d(st + R.offB + i * B_TILE, &mB, b.b_col[i] + kb * BK, brow, &full[s]);
        }
      }
    } else {
      // ---- per-vertex metadata of this CTA's columns, meanwhile (lanes 1..31) ----
      for (int r = (warp - 2) * 31 + lane - 1; r < COLS; r += 8 * 31) {
        const int p = p0 + c_own + r;
        if (p < row_hi) load_meta(D, p, epi_needs_children<E>(), s_meta[r]);
      }
    }
    __syncwarp();
    // ---- stage all accumulators in shared memory: xs[a][col][unit] ----
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    ptx::griddep_wait();                               // (already satisfied: orders the epilogue's reads)
    if (D.trace && threadIdx.x == 64) s_tr[1] = gtime();
    const int qd = warp & 3, grp = (warp - 2) >> 2;
    const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16);
    for (int a = 0; a < R.nacc; ++a) {
#pragma unroll
      for (int c0 = grp * 32; c0 < grp * 32 + 32; c0 += 8) {
        float v[8];
        ptx::tmem_ld<8>(tq + a * NT + c0, v);
        if (P.npair > 1) {                               // split mode: main + corrections (fp32, RN)
          float w[8];
          ptx::tmem_ld<8>(tq + (a + R.nacc) * NT + c0, w);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] += w[i];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) xs[((size_t)a * NT + c0 + i) * 128 + qd * 32 + lane] = v[i];
      }
    }
  }
  ptx::tc_fence_before();
  if constexpr (CL > 1) cluster_sync_all();
  else __syncthreads();
  // ---- fused cell epilogue: thread -> (4 consecutive units, columns) ----
  if (warp >= 2) {
    const int t = threadIdx.x - 64;                    // 0..255
    const int uq = t & 31, cg = t >> 5;                // unit quad, column group
    const int j = m0 + uq * 4;
    const UnitC<4> uc = (epi_uses_bias<E>() && j < units) ? load_unit<4>(D, j, epi_is_lstm<E>()) : UnitC<4>{};
    const uint32_t xs_base = ptx::smem_u32(xs) + (uint32_t)(uq * 4) * 4u;
    constexpr int CPT = (COLS + 7) / 8;                // columns per thread (CL = 16: 4 columns, half the threads)
    constexpr int CH = epi_needs_children<E>() ? 1 : (CPT < 4 ? CPT : 4);
    // children per vertex the epilogue state is sized for
    constexpr int NM = E == EPI_LSTM_FWD ? NACC - 3 : (E == EPI_LSTM_BWD || E == EPI_LSTM_BWD_DAG) ? NACC - 1 : 1;
#pragma unroll 1
    for (int i0 = 0; i0 < CPT; i0 += CH) {
      FV<4> acc[CH][NACC];
      typename EpiK<E>::template In<4, NM> in[CH];
      bool ok[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {                   // gather accumulators + all loads first ...
        const int r = cg + 8 * (i0 + i);               // own column index
        const int c = c_own + r;                       // column in the task tile
        const int p = p0 + c;
        ok[i] = r < COLS && j < units && p < row_hi && row_active<E>(D, p, s_meta[r].xrow);
        if (!ok[i]) continue;
#pragma unroll
        for (int e = 0; e < NACC; ++e) {
          float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int q = 0; q < CL; ++q) {
            const int ai = P.comb[e][q];
            if (ai < 0) continue;
            float4 x;
            if constexpr (CL > 1) x = ld_dsmem4(mapa_rank(xs_base + (uint32_t)((ai * NT + c) * 128) * 4u, q));
            else x = *reinterpret_cast<const float4*>(xs + (size_t)(ai * NT + c) * 128 + uq * 4);
            sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
          }
          acc[i][e].v[0] = sum.x; acc[i][e].v[1] = sum.y; acc[i][e].v[2] = sum.z; acc[i][e].v[3] = sum.w;
        }
        EpiK<E>::template load<4, NM>(D, j, s_meta[r], in[i]);
      }
      if constexpr (epi_is_level<E>()) {
        if (D.unfused) {                               // ablation: raw accumulators only
#pragma unroll
          for (int i = 0; i < CH; ++i)
            if (ok[i]) store_raw<4>(D, j, s_meta[cg + 8 * (i0 + i)].p, acc[i], NACC);
          continue;
        }
      }
#pragma unroll
      for (int i = 0; i < CH; ++i)                     // ... then the math and the stores
        if (ok[i]) EpiK<E>::template store<OpT, 4, NM>(D, j, s_meta[cg + 8 * (i0 + i)], acc[i], in[i], uc);
    }
  }
  if constexpr (CL > 1) cluster_sync_all();            // remote reads done before smem is released
  ptx::tc_fence_before();
  __syncthreads();
  if (D.trace && threadIdx.x == 0) {
    const unsigned long long at = 8 + 8 * atomicAdd(D.trace, 1ull);
    if (at + 8 < (4u << 20) / 8) {
      D.trace[at] = 100 * CL + E; D.trace[at + 1] = blockIdx.x + 1000ull * blockIdx.y; D.trace[at + 2] = row_lo;
      D.trace[at + 3] = s_tr[0]; D.trace[at + 4] = s_tr[2]; D.trace[at + 5] = s_tr[1]; D.trace[at + 6] = gtime();
      D.trace[at + 7] = row_hi;
    }
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------------------------
constexpr int T2_TILE = 2 * 64 * 64 * 2;   // 16 KB: 128 MN x 64 K, two 64x64 TMA boxes

__device__ __forceinline__ bool kb_has_x(const Dev& D, int r0) {
  const int r1 = min(r0 + 63, D.V - 1);
  return D.tile_x[r0 >> 6] || D.tile_x[r1 >> 6];
}

__global__ void __launch_bounds__(kThreads, 1)
k_tc_typeII(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, Dev D, PlanII P,
            float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = P.stages;
  const int STAGE = 2 * T2_TILE * P.planes;            // A then B, each planes x (128 MN x 64 K)
  const int offBp = T2_TILE * P.planes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int* s_count = reinterpret_cast<int*>(tmem_slot + 1);
  int& s_main = s_count[1];                           // the main / correction accumulator was written
  int& s_corr = s_count[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * 128, z = blockIdx.z;
  int nkb_total = 0;
  for (int i = 0; i < P.nseg; ++i) nkb_total += cdiv(P.s[i].k_hi - P.s[i].k_lo, 64);
  const int per = cdiv(nkb_total, P.split);
  const int g_lo = z * per, g_hi = min(nkb_total, g_lo + per);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
    *s_count = 0;
  }
  if (warp == 1) ptx::tmem_alloc<256>(tmem_slot);      // [0,128): main, [128,256): split-mode corrections
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) { ptx::tma_prefetch(&mA); ptx::tma_prefetch(&mB); }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(128, 128, 1, 1);
      int step = 0, g = 0;
      uint32_t wrote = 0;                              // accumulators initialised (bit 0 main, bit 1 corr)
      for (int si = 0; si < P.nseg; ++si) {
        const SegT2 sg = P.s[si];
        const int nkb = cdiv(sg.k_hi - sg.k_lo, 64);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          if (g < g_lo || g >= g_hi) continue;
          if (sg.skip_no_x && !kb_has_x(D, sg.k_lo + kb * 64)) continue;
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&full[s], ph);
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(smem + s * STAGE);
          const uint32_t b0 = a0 + offBp;
          constexpr int PS[6] = {0, 0, 1, 0, 1, 2}, PT[6] = {0, 1, 0, 2, 1, 0};
          for (int pr = 0; pr < (P.planes > 1 ? 6 : 1); ++pr) {
            const uint32_t a = a0 + PS[pr] * T2_TILE, b = b0 + PT[pr] * T2_TILE;
            const uint32_t ac = pr > 0 ? 1u : 0u;        // split mode: corrections in their own accumulator
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::mma_bf16(tmem + ac * 128, ptx::sdesc_sw128(a + kk * 2048, 8192, 1024),
                            ptx::sdesc_sw128(b + kk * 2048, 8192, 1024), idesc, ((wrote >> ac) & 1u) | (kk > 0 ? 1u : 0u));
            wrote |= 1u << ac;
          }
          ptx::mma_commit(&empty[s]);
          ++step;
        }
      }
      *s_count = step;
      s_main = wrote & 1u;
      s_corr = (wrote >> 1) & 1u;
      ptx::mma_commit(done);
    }
    __syncwarp();
  } else {
    if (lane == 0) {
      // ---- TMA issue, one warp per pipeline stage (warp 2 + s owns stage s) ----
      const int w = warp - 2;
      int step = 0, g = 0;
      for (int si = 0; si < P.nseg; ++si) {
        const SegT2 sg = P.s[si];
        const int nkb = cdiv(sg.k_hi - sg.k_lo, 64);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          if (g < g_lo || g >= g_hi) continue;
          const int r0 = sg.k_lo + kb * 64;
          if (sg.skip_no_x && !kb_has_x(D, r0)) continue;
          if (step % S == w) {
            const int s = step % S;
            const uint32_t ph = (step / S) & 1;
            if (step >= S) ptx::mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * STAGE;
            ptx::mbar_arrive_expect_tx(&full[s], STAGE);
            for (int q = 0; q < P.planes; ++q) {
              const int ra = r0 + q * P.vp;
              uint8_t* sa = st + q * T2_TILE;
              uint8_t* sb = st + offBp + q * T2_TILE;
              ptx::tma_load_2d(sa, &mA, sg.a_col + m0, ra, &full[s]);
              ptx::tma_load_2d(sa + T2_TILE / 2, &mA, sg.a_col + m0 + 64, ra, &full[s]);
              ptx::tma_load_2d(sb, &mB, sg.b_col + n0, ra, &full[s]);
              ptx::tma_load_2d(sb + T2_TILE / 2, &mB, sg.b_col + n0 + 64, ra, &full[s]);
            }
          }
          ++step;
        }
      }
    }
    __syncwarp();
    if (warp < 6) {
      ptx::mbar_wait(done, 0);
      ptx::tc_fence_after();
      const int qd = warp & 3;
      const int m = m0 + qd * 32 + lane;
      const bool any = *s_count > 0;
      float* o = out + (size_t)z * P.split_stride;
      const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16);
      for (int c = 0; c < 128; c += 16) {
        float v[16];
        ptx::tmem_ld16(tq + c, v);
        if (!s_main) {                                 // (a split-K slot with correction blocks only)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (s_corr) {                                  // split mode: main + corrections (fp32, RN)
          float w[16];
          ptx::tmem_ld16(tq + 128 + c, w);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += w[i];
        }
        if (m < P.M) {
          for (int i = 0; i < 16; ++i) {
            const int n = n0 + c + i;
            if (n < P.Ncols) {
              const float x = any ? v[i] : 0.f;
              float* dst = o + (size_t)m * P.ldo + n;
              *dst = P.accum ? *dst + x : x;              // accum: stream-ordered launches, split 1
            }
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tmem);
  }
}

// =====================================================================================
// host side
// =====================================================================================
struct TcState {
  // K-major A (weights, box 64 x 128), K-major B (arenas, box 64 x NT), MN-major (box 64 x 64)
  CUtensorMap A[5];
  CUtensorMap B_hk, B_xp, B_dz;
  CUtensorMap M_dz, M_hk, M_xp;
  bool use_simt = false;
  bool mono = false;            // CAVS_TC_MONO=1: one CTA per 128-unit block for the levels too
  PersistState* ps = nullptr;   // persistent weight-stationary level kernels (persist.cu), if the shape admits
  GemmState* gs = nullptr;      // row-tiled x-projection / dX GEMMs (gemm.cu)
  LazyState* ls = nullptr;      // stream-K lazy weight-gradient GEMMs (lazy.cu)
  RowsState* rs = nullptr;      // row-tiled level GEMMs for large tasks when the persistent path is off (rows.cu)
  RowsState* rx = nullptr;      // the row-tiled kernel for the x-projection / dX (= rs, or its own state)
  int rows_min_tiles = 64;      // a task uses the row-tiled kernel from this many tiles on
  // FP32 split mode (bf16x3 operands): rows between the planes of each A map (the weight copy's
  // row count) and of the arenas (Vp); 0 = plain bf16
  int split = 0;
  int prow[5] = {0, 0, 0, 0, 0};
  int vp = 0;
  int num_sms = 148;
  int ksl_force = 0;            // CAVS_TC_KSL=1|2|4: K slices per gate rank of the per-task kernels (0: by size)
  // grouped-stage maps (PlanT::kpb): 4-D {64 k, rows, k-block, plane} views of the same tensors, one per
  // kpb in {1, 2, 4} (the box covers kpb k-blocks x all planes); grp = 0: CAVS_TC_GROUP=0 (legacy maps)
  bool grp = false;
  CUtensorMap A4[5][3], B4_hk[3], B4_xp[3], B4_dz[3];
  std::string info;
};

// The launch's plane pairs (FP32 split mode: six products a_s b_t, s + t <= 2, of the bf16x3
// operands; PlanT::npair) for a plan whose A tiles come from A maps ia0 / ia1.
static PlanT pl(const TcState* t, PlanT P, int ia0, int ia1) {
  P.npair = t->split ? 6 : 1;
  P.a_prow[0] = t->split ? t->prow[ia0] : 0;
  P.a_prow[1] = t->split ? t->prow[ia1] : 0;
  P.b_prow = t->split ? t->vp : 0;
  return P;
}
// Type II in the split mode: every segment becomes the six plane-pair segments (rows of plane q of
// an arena start q * Vp rows after plane 0: the MN-major maps span all three planes)
static PlanII pl2(const TcState* t, PlanII P) {
  P.planes = t->split ? 3 : 1;
  P.vp = t->vp;
  return P;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool encode(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_elems,
                   uint32_t box_cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 4-D view {64 k, rows, k-block, plane} of a row-major [planes x rows x K] bf16 tensor (plane q
// plane_rows rows after plane 0), box {64, box_rows, kpb, np}: one box = kpb k-block tiles of box_rows
// rows in every plane, smem order [plane][k-block][row][64] (each tile SW128, K-major)
static bool encode4(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint64_t np, uint64_t plane_rows,
                    uint32_t box_rows, uint32_t kpb) {
  cuuint64_t dims[4] = {64, rows, K / 64, np};
  cuuint64_t strides[3] = {K * 2, 128, plane_rows * K * 2};
  cuuint32_t box[4] = {64, box_rows, kpb, (cuuint32_t)np};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// the grouped-stage map of a legacy map of this context (nullptr: none)
static thread_local const TcState* g_tc = nullptr;
static const CUtensorMap* map4(const CUtensorMap* m, int kidx) {
  const TcState* t = g_tc;
  if (!t || !t->grp) return nullptr;
  for (int i = 0; i < 5; ++i)
    if (m == &t->A[i]) return &t->A4[i][kidx];
  if (m == &t->B_hk) return &t->B4_hk[kidx];
  if (m == &t->B_xp) return &t->B4_xp[kidx];
  if (m == &t->B_dz) return &t->B4_dz[kidx];
  return nullptr;
}

cavs_status tc_init(const Dev& D, int max_vertices, TcState** out, std::string* err) {
  TcState* t = new TcState();
  const char* env = std::getenv("CAVS_BF16_SIMT");
  t->use_simt = env && env[0] == '1';
  const char* mono = std::getenv("CAVS_TC_MONO");
  t->mono = mono && mono[0] == '1';
  if (const char* k = std::getenv("CAVS_TC_KSL")) t->ksl_force = std::atoi(k);
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      *err = "cuTensorMapEncodeTiled unavailable";
      delete t;
      return CAVS_E_CUDA;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const uint64_t h = D.h, d = D.d, N = D.N, Vp = (uint64_t)max_vertices + kPadRows;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const uint64_t G = lstm ? 3 + N : 1;
  // FP32 split mode: each map spans the three bf16 planes (plane-major: plane q starts q x the
  // plane's row count after plane 0), the plans add the plane row offsets (pl / pl2)
  const uint64_t np = D.split ? 3 : 1;
  t->split = D.split;
  t->vp = (int)Vp;
  bool ok = true;
  if (lstm) {
    ok &= encode(&t->A[0], D.Wa, h, np * 4 * h, h, BK, 128);          // U4   [4h x h]
    ok &= encode(&t->A[1], D.Wb, d, np * 4 * h, d, BK, 128);          // W4   [4h x d]
    ok &= encode(&t->A[2], D.Wc, 3 * h, np * h, 3 * h, BK, 128);      // UTiou[h x 3h]
    ok &= encode(&t->A[3], D.Wd, h, np * h, h, BK, 128);              // UTf  [h x h]
    ok &= encode(&t->A[4], D.We, G * h, np * d, G * h, BK, 128);      // WT   [d x G h]
    const int pr[5] = {(int)(4 * h), (int)(4 * h), (int)h, (int)h, (int)d};
    for (int i = 0; i < 5; ++i) t->prow[i] = pr[i];
  } else {
    ok &= encode(&t->A[0], D.Wa, 2 * h, np * h, 2 * h, BK, 128);      // Wc   [h x 2h]
    ok &= encode(&t->A[1], D.Wb, d, np * h, d, BK, 128);              // Wx   [h x d]
    ok &= encode(&t->A[2], D.Wc, h, np * 2 * h, h, BK, 128);          // WcT  [2h x h]
    t->A[3] = t->A[2];
    ok &= encode(&t->A[4], D.We, h, np * d, h, BK, 128);              // WxT  [d x h]
    const int pr[5] = {(int)h, (int)h, (int)(2 * h), (int)(2 * h), (int)d};
    for (int i = 0; i < 5; ++i) t->prow[i] = pr[i];
  }
  ok &= encode(&t->B_hk, D.Hk, N * h, np * Vp, N * h, BK, NT);
  ok &= encode(&t->B_xp, D.Xp, d, np * Vp, d, BK, NT);
  ok &= encode(&t->B_dz, D.dZ, G * h, np * Vp, G * h, BK, NT);
  ok &= encode(&t->M_dz, D.dZ, G * h, np * Vp, G * h, 64, 64);
  ok &= encode(&t->M_hk, D.Hk, N * h, np * Vp, N * h, 64, 64);
  ok &= encode(&t->M_xp, D.Xp, d, np * Vp, d, 64, 64);
  {
    // opt-in (CAVS_TC_GROUP=1): measured slower than the per-k-block boxes issued by one warp per stage
    // (cfg4 h = 1024 155.8k vs 157.2k, fp32 113.4k vs 120.7k samples/s; profiles/r02_ablations.md)
    const char* ge = std::getenv("CAVS_TC_GROUP");
    t->grp = ge && ge[0] == '1';
    // A maps: (base, K = row width, rows per plane) as the 2-D maps above
    const void* ab[5] = {D.Wa, D.Wb, D.Wc, lstm ? D.Wd : D.Wc, D.We};
    uint64_t ak[5], am[5];
    if (lstm) {
      const uint64_t k5[5] = {h, d, 3 * h, h, G * h}, m5[5] = {4 * h, 4 * h, h, h, d};
      for (int i = 0; i < 5; ++i) { ak[i] = k5[i]; am[i] = m5[i]; }
    } else {
      const uint64_t k5[5] = {2 * h, d, h, h, h}, m5[5] = {h, h, 2 * h, 2 * h, d};
      for (int i = 0; i < 5; ++i) { ak[i] = k5[i]; am[i] = m5[i]; }
    }
    for (int kx = 0; kx < 3 && t->grp; ++kx) {
      const uint32_t kpb = 1u << kx;
      for (int i = 0; i < 5; ++i) t->grp &= encode4(&t->A4[i][kx], ab[i], ak[i], am[i], np, am[i], 128, kpb);
      t->grp &= encode4(&t->B4_hk[kx], D.Hk, N * h, Vp, np, Vp, NT, kpb);
      t->grp &= encode4(&t->B4_xp[kx], D.Xp, d, Vp, np, Vp, NT, kpb);
      t->grp &= encode4(&t->B4_dz[kx], D.dZ, G * h, Vp, np, Vp, NT, kpb);
    }
  }
  if (!ok) {
    *err = "cuTensorMapEncodeTiled failed";
    delete t;
    return CAVS_E_CUDA;
  }
  if (D.split) {
    // FP32 mode on the tensor cores: the per-task type-I kernels (gate-split clusters, monolithic
    // x-projection / dX) and the split-K type-II lazy GEMMs, six bf16 MMAs per fp32 product
    t->use_simt = false;
    t->mono = false;
    t->info = "levels: FP32 on tcgen05 (bf16x3 split operands, 6 MMAs per product), per-task launches; "
              "lazy: split-K tcgen05 + pack";
    *out = t;
    return CAVS_OK;
  }
  if (!t->use_simt) t->gs = gemm_init(D, max_vertices);
  if (!t->use_simt) t->ls = lazy_init(D, max_vertices);
  if (t->use_simt) t->info = "levels: SIMT FFMA (CAVS_BF16_SIMT=1)";
  else if (t->mono) t->info = "levels: per-task tcgen05, monolithic CTAs (CAVS_TC_MONO=1)";
  else if (D.unfused || D.stream_x) {
    t->info = std::string("levels: per-task tcgen05 launches (ablation: ") +
              (D.unfused ? "unfused cell epilogues" : "") + (D.unfused && D.stream_x ? ", " : "") +
              (D.stream_x ? "streamed x-projection" : "") + ")";
  } else {
    std::string why;
    t->ps = persist_init(D, max_vertices, &why);
    t->info = t->ps ? "levels: " + persist_describe(t->ps)
                    : "levels: per-task tcgen05 launches (persistent path unavailable: " + why + ")";
    if (!t->ps) {
      t->rs = rows_init(D, max_vertices);
      const char* mt = std::getenv("CAVS_ROWS_MIN_TILES");
      if (mt) t->rows_min_tiles = std::atoi(mt);
      if (t->rs) t->info += "; large tasks: row-tiled tcgen05 (>= " + std::to_string(t->rows_min_tiles) + " tiles" +
                            (rows_pair(t->rs) == 2 ? ", CTA pairs)" : ")");
    }
    t->rx = t->rs ? t->rs : rows_init(D, max_vertices);
    if (t->rx && !rows_xd(t->rx)) {
      if (t->rx != t->rs) rows_destroy(t->rx);
      t->rx = nullptr;
    }
    if (t->rx) t->info += "; x-projection / dX: row-tiled tcgen05";
  }
  t->info += D.lazy_off ? "; lazy batching OFF (ablation: per-task weight-gradient GEMMs)"
                        : t->ls ? "; lazy: stream-K tcgen05 (one launch)" : "; lazy: split-K tcgen05 + pack";
  *out = t;
  return CAVS_OK;
}

std::string tc_describe(const TcState* tc) { return tc ? tc->info : std::string("levels: FP32 FFMA"); }

int tc_clusters(const TcState* tc) { return tc && tc->ps ? persist_clusters(tc->ps) : 0; }
bool tc_sync_free_capable(const TcState* tc) {
  return tc && tc->ps && !persist_has_kbwd(tc->ps) && tc->ls && tc->gs && !tc->use_simt && !tc->mono;
}

void tc_destroy(TcState* tc) {
  if (tc && tc->ps) persist_destroy(tc->ps);
  if (tc && tc->gs) gemm_destroy(tc->gs);
  if (tc && tc->ls) lazy_destroy(tc->ls);
  if (tc && tc->rx && tc->rx != tc->rs) rows_destroy(tc->rx);
  if (tc && tc->rs) rows_destroy(tc->rs);
  delete tc;
}

// ---- type-I plans ---------------------------------------------------------------------
static PlanT plan_empty() {
  PlanT P{};
  P.npair = 1;
  for (int e = 0; e < 8; ++e)
    for (int r = 0; r < kClMax; ++r) P.comb[e][r] = -1;
  return P;
}

static Bundle bundle(int map_a, int nA, const int* a_rows, int a_col0, int nB, const int* b_cols, int nk) {
  Bundle b{};
  b.map_a = map_a; b.nA = nA;
  for (int i = 0; i < nA; ++i) b.a_row[i] = a_rows[i];
  b.a_col0 = a_col0;
  b.nB = nB;
  for (int i = 0; i < nB; ++i) b.b_col[i] = b_cols[i];
  b.nk = nk;
  return b;
}
static void add_mma(Bundle& b, int a, int bt, int acc) {
  b.mma_a[b.nmma] = a; b.mma_b[b.nmma] = bt; b.mma_acc[b.nmma] = acc; ++b.nmma;
}

static int plan_finalize(PlanT& P, int CL) {
  int pipe = 0, xs = 0;
  const int np = P.npair > 1 ? 3 : 1;                  // split mode: three planes of every tile per stage
  if (P.kpb > 0) {                                     // grouped stages: the largest kpb with >= 2 stages
    int per = 0, maxnk = 1;
    for (int r = 0; r < CL; ++r) {
      const RankPlan& R = P.r[r];
      int maxA = 1, maxB = 1;
      for (int i = 0; i < R.nb; ++i) {
        maxA = std::max(maxA, R.b[i].nA); maxB = std::max(maxB, R.b[i].nB); maxnk = std::max(maxnk, R.b[i].nk);
      }
      per = std::max(per, np * (maxA * A_TILE + maxB * B_TILE));
    }
    int kpb = 4;
    while (kpb > 1 && (2 * kpb * per > kSmemBudget || kpb > maxnk)) kpb /= 2;
    P.kpb = kpb;
  }
  const int kg = P.kpb > 0 ? P.kpb : 1;
  for (int r = 0; r < CL; ++r) {
    RankPlan& R = P.r[r];
    int maxA = 1, maxB = 1;
    for (int i = 0; i < R.nb; ++i) { maxA = std::max(maxA, R.b[i].nA); maxB = std::max(maxB, R.b[i].nB); }
    R.offB = kg * np * maxA * A_TILE;
    R.stage_bytes = R.offB + kg * np * maxB * B_TILE;
    R.stages = std::max(1, std::min(6, kSmemBudget / R.stage_bytes));
    pipe = std::max(pipe, R.stages * R.stage_bytes);
    xs = std::max(xs, R.nacc * NT * 128 * 4);
  }
  P.bar_off = (std::max(pipe, xs) + 1023) & ~1023;
  return 1024 + P.bar_off + 2 * 6 * 8 + 16 + 64;
}

// K range [0, nkb) k-blocks split over the cluster ranks (contiguous, balanced).
static void ksplit(int nkb, int r, int* kb0, int* nk) {
  const int q = nkb / kCluster, rem = nkb % kCluster;
  *kb0 = r * q + std::min(r, rem);
  *nk = q + (r < rem ? 1 : 0);
}

// gate split: every rank takes its K share of (A rows a_row, A col a_col, B col b_col) -> slot e
static void gs_add_ksplit(PlanT& P, int map_a, int a_row, int a_col, int b_col, int K, int e) {
  const int nkb = K / BK;
  for (int r = 0; r < kCluster; ++r) {
    int kb0, nk;
    ksplit(nkb, r, &kb0, &nk);
    if (nk == 0) continue;
    RankPlan& R = P.r[r];
    const int bc = b_col + kb0 * BK;
    Bundle b = bundle(map_a, 1, &a_row, a_col + kb0 * BK, 1, &bc, nk);
    add_mma(b, 0, 0, R.nacc);
    R.b[R.nb++] = b;
    P.comb[e][r] = R.nacc++;
  }
}

// K-sliced gate split (small tasks: spread F's weight stream over more SMs): rank g of a kCluster
// gate-split plan becomes ranks g ksl + q, q < ksl, each running k-blocks [q nk / ksl, (q + 1) nk / ksl)
// of every bundle of g into its own accumulators; the epilogue sums the slices like the gate ranks
// (comb).  nullopt-like: returns false if some bundle has fewer than ksl k-blocks.
static bool kslice(const PlanT& G, int ksl, PlanT* out) {
  PlanT P = G;
  for (int g = 0; g < kCluster; ++g)
    for (int q = 0; q < ksl; ++q) {
      RankPlan R = G.r[g];
      for (int bi = 0; bi < R.nb; ++bi) {
        Bundle& b = R.b[bi];
        if (b.nk < ksl) return false;
        const int k0 = (b.nk * q) / ksl, k1 = (b.nk * (q + 1)) / ksl;
        b.a_col0 += k0 * BK;
        for (int i = 0; i < b.nB; ++i) b.b_col[i] += k0 * BK;
        b.nk = k1 - k0;
      }
      P.r[g * ksl + q] = R;
    }
  for (int e = 0; e < 8; ++e)
    for (int g = 0; g < kCluster; ++g)
      for (int q = 0; q < ksl; ++q) P.comb[e][g * ksl + q] = G.comb[e][g];
  *out = P;
  return true;
}

// ---- Tree-LSTM, forward task: gate g over every child slot (U h~ = sum_k U h_k) ----
static PlanT mono_lstm_fwd(int h, int N) {
  PlanT P = plan_empty();
  const int rows[4] = {0, h, 2 * h, 3 * h};
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = k * h;
  Bundle b = bundle(0, 4, rows, 0, N, cols, h / BK);
  for (int g = 0; g < 3; ++g)
    for (int k = 0; k < N; ++k) add_mma(b, g, k, g);
  for (int k = 0; k < N; ++k) add_mma(b, 3, k, 3 + k);
  RankPlan& R = P.r[0];
  R.b[0] = b; R.nb = 1; R.nacc = 3 + N;
  for (int e = 0; e < 3 + N; ++e) P.comb[e][0] = e;
  return P;
}
static PlanT gs_lstm_fwd(int h, int N) {
  PlanT P = plan_empty();
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = k * h;
  for (int g = 0; g < 4; ++g) {
    const int row = g * h;
    Bundle b = bundle(0, 1, &row, 0, N, cols, h / BK);
    RankPlan& R = P.r[g];
    if (g < 3) {
      for (int k = 0; k < N; ++k) add_mma(b, 0, k, 0);
      R.nacc = 1;
      P.comb[g][g] = 0;
    } else {
      for (int k = 0; k < N; ++k) { add_mma(b, 0, k, k); P.comb[3 + k][3] = k; }
      R.nacc = N;
    }
    R.b[0] = b; R.nb = 1;
  }
  return P;
}
// ---- Tree-LSTM eager pull projection: gates of W4 over Xp ----
static PlanT mono_lstm_xproj(int h, int d) {
  PlanT P = plan_empty();
  const int rows[4] = {0, h, 2 * h, 3 * h};
  const int zero = 0;
  Bundle b = bundle(0, 4, rows, 0, 1, &zero, d / BK);
  for (int g = 0; g < 4; ++g) { add_mma(b, g, 0, g); P.comb[g][0] = g; }
  P.r[0].b[0] = b; P.r[0].nb = 1; P.r[0].nacc = 4;
  return P;
}
// gate-split variant (split mode: the four gates' A tiles x three planes do not fit one stage)
static PlanT gs_lstm_xproj(int h, int d) {
  PlanT P = plan_empty();
  const int zero = 0;
  for (int g = 0; g < 4; ++g) {
    const int row = g * h;
    Bundle b = bundle(0, 1, &row, 0, 1, &zero, d / BK);
    add_mma(b, 0, 0, 0);
    P.r[g].b[0] = b; P.r[g].nb = 1; P.r[g].nacc = 1;
    P.comb[g][g] = 0;
  }
  return P;
}
// ---- Tree-LSTM backward task: slot 0 = U_iou^T dz_iou, slot 1+k = U_f^T dz_fk ----
static PlanT mono_lstm_bwd(int h, int N) {
  PlanT P = plan_empty();
  RankPlan& R = P.r[0];
  const int zero = 0;
  R.b[0] = bundle(0, 1, &zero, 0, 1, &zero, 3 * h / BK);
  add_mma(R.b[0], 0, 0, 0);
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = (3 + k) * h;
  R.b[1] = bundle(1, 1, &zero, 0, N, cols, h / BK);
  for (int k = 0; k < N; ++k) add_mma(R.b[1], 0, k, 1 + k);
  R.nb = 2; R.nacc = 1 + N;
  for (int e = 0; e < 1 + N; ++e) P.comb[e][0] = e;
  return P;
}
static PlanT gs_lstm_bwd(int h, int N) {
  PlanT P = plan_empty();
  const int zero = 0;
  for (int g = 0; g < 3; ++g) {
    const int bc = g * h;
    Bundle b = bundle(0, 1, &zero, g * h, 1, &bc, h / BK);
    add_mma(b, 0, 0, 0);
    P.r[g].b[0] = b; P.r[g].nb = 1; P.r[g].nacc = 1;
    P.comb[0][g] = 0;
  }
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = (3 + k) * h;
  Bundle b = bundle(1, 1, &zero, 0, N, cols, h / BK);
  for (int k = 0; k < N; ++k) { add_mma(b, 0, k, k); P.comb[1 + k][3] = k; }
  P.r[3].b[0] = b; P.r[3].nb = 1; P.r[3].nacc = N;
  return P;
}
// ---- Tree-LSTM dX: W^T over dZ (the f blocks of W^T all hold W_f) ----
static PlanT mono_lstm_dx(int h, int N) {
  PlanT P = plan_empty();
  const int zero = 0;
  Bundle b = bundle(0, 1, &zero, 0, 1, &zero, (3 + N) * h / BK);
  add_mma(b, 0, 0, 0);
  P.r[0].b[0] = b; P.r[0].nb = 1; P.r[0].nacc = 1;
  P.comb[0][0] = 0;
  return P;
}
// ---- single-rank plan: slot e = A rows a_rows[e] x B cols b_cols[e] over K ----
static PlanT mono_one(int K, int e_count, const int* a_rows, const int* b_cols) {
  PlanT P = plan_empty();
  RankPlan& R = P.r[0];
  for (int e = 0; e < e_count; ++e) {
    Bundle b = bundle(0, 1, &a_rows[e], 0, 1, &b_cols[e], K / BK);
    add_mma(b, 0, 0, e);
    R.b[R.nb++] = b;
    P.comb[e][0] = e;
  }
  R.nacc = e_count;
  return P;
}

template <int E, int NACC, int CL, class OpT>
static void launch_level(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b, const Dev& D, PlanT P,
                         int row_lo, int row_hi, int units, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  // grouped stages when this context has the 4-D views of the three maps (kpb chosen by plan_finalize)
  const CUtensorMap *ga0 = map4(&a0, 0), *ga1 = map4(&a1, 0), *gb = map4(&b, 0);
  P.kpb = (ga0 && ga1 && gb) ? 1 : 0;
  const int smem = plan_finalize(P, CL);
  const int kx = P.kpb == 4 ? 2 : P.kpb == 2 ? 1 : 0;
  const CUtensorMap& A0 = P.kpb > 0 ? *map4(&a0, kx) : a0;
  const CUtensorMap& A1 = P.kpb > 0 ? *map4(&a1, kx) : a1;
  const CUtensorMap& B0 = P.kpb > 0 ? *map4(&b, kx) : b;
  static int attr_set[kMaxDev] = {};                   // dynamic + static smem must stay <= 227 KB
  const int dv = cur_device();
  if (smem > attr_set[dv]) {
    cudaFuncSetAttribute(k_tc_level<E, NACC, CL, OpT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (CL > 8) cudaFuncSetAttribute(k_tc_level<E, NACC, CL, OpT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_set[dv] = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CL * cdiv(units, 128), cdiv(row_hi - row_lo, NT), 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cudaLaunchAttribute at2[2];
  int na = 0;
  if (CL > 1) at2[na++] = at[0];
  at2[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL: overlap with the previous task
  at2[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  cfg.attrs = at2;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k_tc_level<E, NACC, CL, OpT>, A0, A1, B0, D, P, row_lo, row_hi, units);
}

// per-task dispatch on the arity N (NACC = BASE + N) and the cluster size cl (1: monolithic, 4: gate
// split, 8 / 16: K-sliced gate split, N <= 2)
template <int E, int NACC, class OpT>
static void level_cl(int cl, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b, const Dev& D,
                     const PlanT& P, int lo, int hi, int units, cudaStream_t s) {
  if (cl == 1) launch_level<E, NACC, 1, OpT>(a0, a1, b, D, P, lo, hi, units, s);
  else if (cl == kCluster) launch_level<E, NACC, kCluster, OpT>(a0, a1, b, D, P, lo, hi, units, s);
  else if constexpr (NACC <= 5) {
    if (cl == 8) launch_level<E, NACC, 8, OpT>(a0, a1, b, D, P, lo, hi, units, s);
    else launch_level<E, NACC, 16, OpT>(a0, a1, b, D, P, lo, hi, units, s);
  }
}
template <int E, int BASE, class OpT>
static void level_N(int cl, int N, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b, const Dev& D,
                    const PlanT& P, int lo, int hi, int units, cudaStream_t s) {
  switch (N) {
    case 1: level_cl<E, BASE + 1, OpT>(cl, a0, a1, b, D, P, lo, hi, units, s); break;
    case 2: level_cl<E, BASE + 2, OpT>(cl, a0, a1, b, D, P, lo, hi, units, s); break;
    case 3: level_cl<E, BASE + 3, OpT>(cl, a0, a1, b, D, P, lo, hi, units, s); break;
    default: level_cl<E, BASE + 4, OpT>(cl, a0, a1, b, D, P, lo, hi, units, s); break;
  }
}

// K slices per gate rank for a task of M rows (cluster = kCluster x ksl CTAs per 128-unit block): the
// weight stream of a small task spread over more SMs while every cluster stays resident
static int pick_ksl(const TcState* t, int M, int units) {
  if (t->ksl_force > 0) return t->ksl_force;
  const int nclu = cdiv(units, 128) * cdiv(M, NT);   // clusters of the task
  if (nclu * kCluster * 4 <= t->num_sms && nclu <= 7) return 4;
  if (nclu * kCluster * 2 <= t->num_sms) return 2;
  return 1;
}

// the task's plan and cluster size: gate split (K-sliced for small tasks, arity <= 2) or monolithic
static PlanT gsplan(const TcState* t, const Dev& D, bool gs, const PlanT& G, int M, int units, int* cl) {
  if (!gs) { *cl = 1; return G; }
  int ksl = D.N <= 2 ? pick_ksl(t, M, units) : 1;
  PlanT K;
  while (ksl > 1 && !kslice(G, ksl, &K)) ksl /= 2;
  *cl = kCluster * ksl;
  return ksl > 1 ? K : G;
}

// Streaming ablation: level-0 rows of the x-projection (they finish the leaves) on the main
// stream; the rows of every task above level 0 on the side stream, task t waiting only for its own.
static bool xproj_streamed(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, XStream* xs, Prof& P) {
  const int h = D.h, d = D.d, T = (int)lp.size() - 1;
  if (!D.stream_x || !xs || !xs->s) return false;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int zero = 0;
  const PlanT X = lstm ? mono_lstm_xproj(h, d) : mono_one(d, 1, &zero, &zero);
  auto proj = [&](int lo, int hi, cudaStream_t st) {
    if (lstm) launch_level<EPI_LSTM_XPROJ, 4, 1, __nv_bfloat16>(t->A[1], t->A[1], t->B_xp, D, X, lo, hi, h, st);
    else launch_level<EPI_FC_XPROJ, 1, 1, __nv_bfloat16>(t->A[1], t->A[1], t->B_xp, D, X, lo, hi, h, st);
  };
  while ((int)xs->ev.size() < T) { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); xs->ev.push_back(e); }
  cudaEventRecord(xs->start, s);                     // prep / pull done
  cudaStreamWaitEvent(xs->s, xs->start, 0);
  for (int tt = 1; tt < T; ++tt) {
    proj(lp[tt], lp[tt + 1], xs->s);
    cudaEventRecord(xs->ev[tt], xs->s);
  }
  proj(0, T > 1 ? lp[1] : D.V, s);
  P.count(T);
  return true;
}

template <class OpT>
static void fwd_t(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, Prof& P, XStream* xs) {
  const int skmax = skinny_max(D);
  if (t->use_simt) { simt_forward<__nv_bfloat16>(D, lp, s, P, xs); return; }
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  const bool gs = !t->mono;
  const SegListI Fs = fwd_segments(D);
  const int zero = 0;
  const bool streamed = xproj_streamed(D, t, lp, s, xs, P);
  auto wait_x = [&](int tt) { if (streamed) cudaStreamWaitEvent(s, xs->ev[tt], 0); };
  auto unfused = [&](int epi, int tt) { if (D.unfused) { launch_unfused(D, epi, lp[tt], lp[tt + 1], s); P.count(1); } };
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    // eager pull projection fused with task 0 (large: monolithic CTAs reuse the x tile for 4 gates)
    if (!streamed) {
      if (D.split)
        launch_level<EPI_LSTM_XPROJ, 4, kCluster, OpT>(t->A[1], t->A[1], t->B_xp, D, pl(t, gs_lstm_xproj(h, d), 1, 1),
                                                        0, D.V, h, s);
      else if (!rows_xproj(D, t->rx, s) && !gemm_xproj(D, t->gs, s))
        launch_level<EPI_LSTM_XPROJ, 4, 1, OpT>(t->A[1], t->A[1], t->B_xp, D, pl(t, mono_lstm_xproj(h, d), 1, 1), 0, D.V, h, s);
      P.count(1);
    }
    P.mark(CAVS_PH_FWD_LEVELS, s);
    if (t->ps && !D.dag) { if (T > 1 || D.sync_free) { persist_forward(D, t->ps, T, s); P.count(1); } return; }
    const PlanT F = gs ? gs_lstm_fwd(h, N) : mono_lstm_fwd(h, N);
    for (int tt = 1; tt < T; ++tt) {
      const int M = lp[tt + 1] - lp[tt];
      if (D.dag) { launch_dag_gather(D, lp[tt], lp[tt + 1], s); P.count(1); }
      wait_x(tt);
      if (M <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_FWD, Fs, lp[tt], lp[tt + 1], h, s);
      else if (rows_tiles(t->rs, false, M) >= t->rows_min_tiles && rows_level(D, t->rs, false, lp[tt], lp[tt + 1], s)) {}
      else {
        int cl;
        const PlanT Fk = gsplan(t, D, gs, F, M, h, &cl);
        level_N<EPI_LSTM_FWD, 3, OpT>(cl, N, t->A[0], t->A[0], t->B_hk, D, pl(t, Fk, 0, 0), lp[tt], lp[tt + 1], h, s);
      }
      P.count(1);
      unfused(EPI_LSTM_FWD, tt);
    }
  } else {
    if (!streamed) {
      if (!rows_xproj(D, t->rx, s) && !gemm_xproj(D, t->gs, s))
        launch_level<EPI_FC_XPROJ, 1, 1, OpT>(t->A[1], t->A[1], t->B_xp, D, pl(t, mono_one(d, 1, &zero, &zero), 1, 1), 0, D.V, h, s);
      P.count(1);
    }
    P.mark(CAVS_PH_FWD_LEVELS, s);
    if (t->ps && !D.dag) { if (T > 1 || D.sync_free) { persist_forward(D, t->ps, T, s); P.count(1); } return; }
    PlanT F;
    if (gs) { F = plan_empty(); gs_add_ksplit(F, 0, 0, 0, 0, 2 * h, 0); }
    else F = mono_one(2 * h, 1, &zero, &zero);
    for (int tt = 1; tt < T; ++tt) {
      const int M = lp[tt + 1] - lp[tt];
      if (D.dag) { launch_dag_gather(D, lp[tt], lp[tt + 1], s); P.count(1); }
      wait_x(tt);
      if (M <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_FWD, Fs, lp[tt], lp[tt + 1], h, s);
      else if (rows_tiles(t->rs, false, M) >= t->rows_min_tiles && rows_level(D, t->rs, false, lp[tt], lp[tt + 1], s)) {}
      else if (gs) {
        int cl;
        const PlanT Fk = gsplan(t, D, gs, F, M, h, &cl);
        level_cl<EPI_FC_FWD, 1, OpT>(cl, t->A[0], t->A[0], t->B_hk, D, pl(t, Fk, 0, 0), lp[tt], lp[tt + 1], h, s);
      }
      else launch_level<EPI_FC_FWD, 1, 1, OpT>(t->A[0], t->A[0], t->B_hk, D, pl(t, F, 0, 0), lp[tt], lp[tt + 1], h, s);
      P.count(1);
      unfused(EPI_FC_FWD, tt);
    }
  }
}

static int launch_II(const CUtensorMap& a, const CUtensorMap& b, const Dev& D, PlanII P, float* out,
                     cudaStream_t s) {
  int nkb = 0;
  for (int i = 0; i < P.nseg; ++i) nkb += cdiv(P.s[i].k_hi - P.s[i].k_lo, 64);
  const int tiles = cdiv(P.M, 128) * cdiv(P.Ncols, 128);
  P.split = P.split == 1 ? 1      // forced (per-task ablation launches accumulate in stream order)
            : std::max(1, std::min(std::min(kSplitMax, 148 / std::max(1, tiles)), std::max(1, nkb / 4)));
  if (P.planes < 1) P.planes = 1;
  P.stages = P.planes > 1 ? 2 : 6;
  const int smem = P.stages * 2 * T2_TILE * P.planes + 1024 + 2 * 8 * P.stages + 64;
  static bool attr_done[kMaxDev] = {};
  const int dv = cur_device();
  if (!attr_done[dv]) {
    cudaFuncSetAttribute(k_tc_typeII, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done[dv] = true;
  }
  dim3 grid(cdiv(P.M, 128), cdiv(P.Ncols, 128), P.split);
  k_tc_typeII<<<grid, kThreads, smem, s>>>(a, b, D, P, out);
  return P.split;
}

// pull's adjoint: dX = dZ W
template <class OpT>
static void launch_dx(Dev& D, TcState* t, cudaStream_t s) {
  const int h = D.h, N = D.N, V = D.V, d = D.d;
  const int zero = 0;
  if (rows_dx(D, t->rx, s) || gemm_dx(D, t->gs, s)) return;
  if (D.cell == CAVS_CELL_TREE_LSTM)
    launch_level<EPI_DX, 1, 1, OpT>(t->A[4], t->A[4], t->B_dz, D, pl(t, mono_lstm_dx(h, N), 4, 4), 0, V, d, s);
  else
    launch_level<EPI_DX, 1, 1, OpT>(t->A[4], t->A[4], t->B_dz, D, pl(t, mono_one(h, 1, &zero, &zero), 4, 4), 0, V, d, s);
}

template <class OpT>
static void bwd_t(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, int* split, Prof& P,
                  cudaEvent_t wgrad_ev, cudaEvent_t levels_ev, cudaStream_t dx_s) {
  const int skmax = skinny_max(D);
  split[0] = split[1] = split[2] = 1;
  // dX = dZ W only reads dZ and the weights: on dx_s it overlaps the lazy GEMMs (disjoint outputs);
  // the dx zeroing (usually an early exit) goes with it
  const bool dx_side = dx_s && levels_ev && D.dx && !D.lazy_off && !t->use_simt;
  if (D.dx && D.n_x > 0 && !dx_side) { launch_dx_zero(D, s); P.count(1); }
  if (t->use_simt) {
    simt_backward<__nv_bfloat16>(D, lp, s, P);
    if (levels_ev) cudaEventRecord(levels_ev, s);      // (db after the whole FFMA backward)
    return;
  }
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int G = lstm ? 3 + N : 1;
  const bool gs = !t->mono;
  const SegListI Bs = bwd_segments(D);
  if (D.dag) {
    // DAG batch (NEXT-3): per task, the pull-reduce + dF of its vertices (every parent is in a
    // later task, already done), then the level GEMM whose epilogue only sends the edge gradients
    const PlanT B = lstm ? (gs ? gs_lstm_bwd(h, N) : mono_lstm_bwd(h, N)) : PlanT{};
    PlanT Bfc;
    const int rows[2] = {0, h}, zeros[2] = {0, 0};
    if (!lstm) {
      if (gs) { Bfc = plan_empty(); for (int k = 0; k < 2; ++k) gs_add_ksplit(Bfc, 0, k * h, 0, 0, h, k); }
      else Bfc = mono_one(h, 2, rows, zeros);
    }
    for (int tt = T - 1; tt >= 0; --tt) {
      launch_dag_df(D, lp[tt], lp[tt + 1], s);
      P.count(1);
      if (tt == 0) break;
      const int M = lp[tt + 1] - lp[tt];
      if (lstm) {
        if (M <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_BWD_DAG, Bs, lp[tt], lp[tt + 1], h, s);
        else {
          int cl;
          const PlanT Bk = gsplan(t, D, gs, B, M, h, &cl);
          level_N<EPI_LSTM_BWD_DAG, 1, OpT>(cl, N, t->A[2], t->A[3], t->B_dz, D, pl(t, Bk, 2, 3), lp[tt], lp[tt + 1], h, s);
        }
      } else {
        if (M <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_BWD_DAG, Bs, lp[tt], lp[tt + 1], h, s);
        else if (gs) {
          int cl;
          const PlanT Bk = gsplan(t, D, gs, Bfc, M, h, &cl);
          level_cl<EPI_FC_BWD_DAG, 2, OpT>(cl, t->A[2], t->A[2], t->B_dz, D, pl(t, Bk, 2, 2), lp[tt], lp[tt + 1], h, s);
        }
        else launch_level<EPI_FC_BWD_DAG, 2, 1, OpT>(t->A[2], t->A[2], t->B_dz, D, pl(t, Bfc, 2, 2), lp[tt], lp[tt + 1], h, s);
      }
      P.count(1);
      if (D.unfused) { launch_unfused(D, lstm ? EPI_LSTM_BWD_DAG : EPI_FC_BWD_DAG, lp[tt], lp[tt + 1], s); P.count(1); }
    }
  } else if (t->ps) {
    if (T > 1 || D.sync_free) { persist_backward(D, t->ps, T, s); P.count(1); }
  } else if (lstm) {
    const PlanT B = gs ? gs_lstm_bwd(h, N) : mono_lstm_bwd(h, N);
    for (int tt = T - 1; tt >= 1; --tt) {
      const int M = lp[tt + 1] - lp[tt];
      if (M <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_BWD, Bs, lp[tt], lp[tt + 1], h, s);
      else if (rows_tiles(t->rs, true, M) >= t->rows_min_tiles && rows_level(D, t->rs, true, lp[tt], lp[tt + 1], s)) {}
      else {
        int cl;
        const PlanT Bk = gsplan(t, D, gs, B, M, h, &cl);
        level_N<EPI_LSTM_BWD, 1, OpT>(cl, N, t->A[2], t->A[3], t->B_dz, D, pl(t, Bk, 2, 3), lp[tt], lp[tt + 1], h, s);
      }
      P.count(1);
      if (D.unfused) { launch_unfused(D, EPI_LSTM_BWD, lp[tt], lp[tt + 1], s); P.count(1); }
    }
  } else {
    PlanT B;
    const int rows[2] = {0, h}, zeros[2] = {0, 0};
    if (gs) { B = plan_empty(); for (int k = 0; k < 2; ++k) gs_add_ksplit(B, 0, k * h, 0, 0, h, k); }
    else B = mono_one(h, 2, rows, zeros);
    for (int tt = T - 1; tt >= 1; --tt) {
      const int M = lp[tt + 1] - lp[tt];
      if (M <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_BWD, Bs, lp[tt], lp[tt + 1], h, s);
      else if (rows_tiles(t->rs, true, M) >= t->rows_min_tiles && rows_level(D, t->rs, true, lp[tt], lp[tt + 1], s)) {}
      else if (gs) {
        int cl;
        const PlanT Bk = gsplan(t, D, gs, B, M, h, &cl);
        level_cl<EPI_FC_BWD, 2, OpT>(cl, t->A[2], t->A[2], t->B_dz, D, pl(t, Bk, 2, 2), lp[tt], lp[tt + 1], h, s);
      }
      else launch_level<EPI_FC_BWD, 2, 1, OpT>(t->A[2], t->A[2], t->B_dz, D, pl(t, B, 2, 2), lp[tt], lp[tt + 1], h, s);
      P.count(1);
      if (D.unfused) { launch_unfused(D, EPI_FC_BWD, lp[tt], lp[tt + 1], s); P.count(1); }
    }
  }
  if (levels_ev) cudaEventRecord(levels_ev, s);      // every dZ row final: db may run beside the lazy GEMMs
  if (dx_side) {
    cudaStreamWaitEvent(dx_s, levels_ev, 0);
    if (D.n_x > 0) { launch_dx_zero(D, dx_s); P.count(1); }
    launch_dx<OpT>(D, t, dx_s);
    P.count(1);
  }
  P.mark(CAVS_PH_LAZY, s);
  // ---- lazy batching of the parameter gradients ----
  const LazyLayout Z = lazy_layout(D);
  float* u4 = D.lazy + Z.u4;
  float* uf = D.lazy + Z.uf;
  float* w = D.lazy + Z.w;
  const int lp1 = D.lp1, V = D.V;
  const int zero = 0;
  if (D.lazy_off) {
    // ablation "lazy batching off": the weight gradients as separate GEMMs per task over
    // that task's rows only (what Alg. 1's per-task backward would issue), accumulated in stream
    // order into one slot (split 1; deterministic), then packed like the split-K fallback
    const int Tn = (int)lp.size() - 1;
    for (int tt = 0; tt < Tn; ++tt) {
      const int lo = lp[tt], hi = lp[tt + 1];
      const int acc = tt > 0 ? 1 : 0;
      // dZ viewed with `hi` rows: the TMA zero-fills the last k-block's rows of the next task
      CUtensorMap mdz;
      encode(&mdz, D.dZ, (uint64_t)G * h, (uint64_t)hi, (uint64_t)G * h, 64, 64);
      if (lstm) {
        PlanII A{};                                     // dU_iou, dU_f: parents only (t >= 1)
        A.nseg = N; A.split = 1; A.accum = acc > 0 && tt > 1 ? 1 : 0;
        for (int k = 0; k < N; ++k) A.s[k] = SegT2{0, k * h, lo, tt >= 1 ? hi : lo, 0};
        A.M = 3 * h; A.Ncols = h; A.ldo = h; A.split_stride = Z.su4;
        PlanII Bf = A;
        for (int k = 0; k < N; ++k) Bf.s[k] = SegT2{(3 + k) * h, k * h, lo, tt >= 1 ? hi : lo, 0};
        Bf.M = h; Bf.Ncols = h; Bf.ldo = h; Bf.split_stride = Z.suf;
        if (tt >= 1) { launch_II(mdz, t->M_hk, D, pl2(t, A), u4, s); launch_II(mdz, t->M_hk, D, pl2(t, Bf), uf, s); P.count(2); }
        PlanII Cw{};                                    // dW over this task's pull records
        Cw.nseg = 1; Cw.split = 1; Cw.accum = acc;
        Cw.s[0] = SegT2{0, 0, lo, hi, 1};
        Cw.M = G * h; Cw.Ncols = d; Cw.ldo = d; Cw.split_stride = Z.sw;
        launch_II(mdz, t->M_xp, D, pl2(t, Cw), w, s); P.count(1);
      } else {
        PlanII A{};
        A.nseg = 1; A.split = 1; A.accum = tt > 1 ? 1 : 0;
        A.s[0] = SegT2{0, 0, lo, hi, 0};
        A.M = h; A.Ncols = 2 * h; A.ldo = 2 * h; A.split_stride = Z.su4;
        if (tt >= 1) { launch_II(mdz, t->M_hk, D, pl2(t, A), u4, s); P.count(1); }
        PlanII Cw{};
        Cw.nseg = 1; Cw.split = 1; Cw.accum = acc;
        Cw.s[0] = SegT2{0, 0, lo, hi, 1};
        Cw.M = h; Cw.Ncols = d; Cw.ldo = d; Cw.split_stride = Z.sw;
        launch_II(mdz, t->M_xp, D, pl2(t, Cw), w, s); P.count(1);
      }
    }
    if (Tn <= 1) {                                      // no internal vertex: dU = 0
      cudaMemsetAsync(u4, 0, sizeof(float) * Z.su4, s);
      if (lstm) cudaMemsetAsync(uf, 0, sizeof(float) * Z.suf, s);
    }
    split[0] = split[1] = split[2] = 1;
  } else if (lazy_grads(D, t->ls, s)) {                // every dU / dW block straight into dparams
    P.count(1);
    split[0] = -1;
    if (wgrad_ev) cudaEventRecord(wgrad_ev, s);        // the weight blocks can be all-reduced from here on
  } else if (lstm) {
    PlanII A{};                                         // dU_iou = sum_k dZ_iou^T H_k  (h~ by linearity)
    A.nseg = N;
    for (int k = 0; k < N; ++k) A.s[k] = SegT2{0, k * h, lp1, V, 0};
    A.M = 3 * h; A.Ncols = h; A.ldo = h; A.split_stride = Z.su4;
    if (lp1 < V) { split[0] = launch_II(t->M_dz, t->M_hk, D, pl2(t, A), u4, s); P.count(1); }
    else cudaMemsetAsync(u4, 0, sizeof(float) * Z.su4, s);
    PlanII Bf{};                                        // dU_f = sum_k dZ_fk^T H_k
    Bf.nseg = N;
    for (int k = 0; k < N; ++k) Bf.s[k] = SegT2{(3 + k) * h, k * h, lp1, V, 0};
    Bf.M = h; Bf.Ncols = h; Bf.ldo = h; Bf.split_stride = Z.suf;
    if (lp1 < V) { split[1] = launch_II(t->M_dz, t->M_hk, D, pl2(t, Bf), uf, s); P.count(1); }
    else cudaMemsetAsync(uf, 0, sizeof(float) * Z.suf, s);
    PlanII Cw{};                                        // dW = dZ^T X over the pull records
    Cw.nseg = 1;
    Cw.s[0] = SegT2{0, 0, 0, V, 1};
    Cw.M = G * h; Cw.Ncols = d; Cw.ldo = d; Cw.split_stride = Z.sw;
    split[2] = launch_II(t->M_dz, t->M_xp, D, pl2(t, Cw), w, s); P.count(1);
  } else {
    PlanII A{};
    A.nseg = 1;
    A.s[0] = SegT2{0, 0, lp1, V, 0};
    A.M = h; A.Ncols = 2 * h; A.ldo = 2 * h; A.split_stride = Z.su4;
    if (lp1 < V) { split[0] = launch_II(t->M_dz, t->M_hk, D, pl2(t, A), u4, s); P.count(1); }
    else cudaMemsetAsync(u4, 0, sizeof(float) * Z.su4, s);
    PlanII Cw{};
    Cw.nseg = 1;
    Cw.s[0] = SegT2{0, 0, 0, V, 1};
    Cw.M = h; Cw.Ncols = d; Cw.ldo = d; Cw.split_stride = Z.sw;
    split[2] = launch_II(t->M_dz, t->M_xp, D, pl2(t, Cw), w, s); P.count(1);
  }
  P.mark(CAVS_PH_DX, s);
  if (D.dx && !dx_side) { launch_dx<OpT>(D, t, s); P.count(1); }
}

void tc_zero_dz_tail(const Dev& D, const TcState* t, cudaStream_t s) {
  if (t->use_simt) return;                            // (the FFMA backward reads no row past V)
  const size_t Gh = (size_t)(D.cell == CAVS_CELL_TREE_LSTM ? 3 + D.N : 1) * D.h;
  for (int q = 0; q < (D.split ? 3 : 1); ++q)
    cudaMemsetAsync(reinterpret_cast<__nv_bfloat16*>(D.dZ) + q * D.ps_dz + (size_t)D.V * Gh, 0, 64 * Gh * 2, s);
}

void tc_forward(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, Prof& P, XStream* xs) {
  g_tc = t;
  if (D.split) fwd_t<S3>(D, t, lp, s, P, xs);
  else fwd_t<__nv_bfloat16>(D, t, lp, s, P, xs);
}

void tc_backward(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, int* split, Prof& P,
                 cudaEvent_t wgrad_ev, cudaEvent_t levels_ev, cudaStream_t dx_s) {
  g_tc = t;
  if (D.split) bwd_t<S3>(D, t, lp, s, split, P, wgrad_ev, levels_ev, dx_s);
  else bwd_t<__nv_bfloat16>(D, t, lp, s, split, P, wgrad_ev, levels_ev, dx_s);
}

}  // namespace cavs
