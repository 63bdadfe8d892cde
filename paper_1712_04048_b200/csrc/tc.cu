// tc.cu — BF16 mode on 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Type I ("level kernel"): one launch per batching task V_t (Alg. 1).
//   D[unit j, vertex n] = sum_k A[j, k] * B[n, k]  with A = weights (K-major, TMA),
//   B = the task's contiguous rows of a position-ordered arena (K-major, TMA) — swap-AB,
//   so the tensor-core M side (128) is the gate units and the small, ragged task size M_t
//   is the N side (tile NT = 64).  Several accumulators per CTA (one per gate) live in
//   TMEM, so the epilogue sees i, o, u, f_1..f_N of the same (unit, vertex) and runs the
//   whole cell (cells.cuh) — gates, activations, child-sum, scatter, push — fused (§3.5
//   "automatic kernel fusion", done by hand).  For the child-sum Tree-LSTM the
//   h~ = sum_k h_k operand is formed in shared memory from the TMA-loaded child slots.
//   Warp roles: w0 TMA producer, w1 TMEM allocator + single-thread MMA issuer,
//   w2..w5 child-sum converters, then epilogue (TMEM -> registers -> cell -> HBM).
// Type II ("lazy GEMM"): the deferred parameter gradients batched over ALL vertices
//   (lazy batching): out[m, n] = sum_p A[p, m] B[p, n] with both operands
//   MN-major straight from the position-ordered arenas, split-K across CTAs.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "cells.cuh"
#include "ptx.cuh"
#include "tc.h"

namespace cavs {

constexpr int NT = 64;                     // task-row tile (MMA N) of type I
constexpr int BK = 64;                     // k-block: one 128-byte swizzle atom of bf16
constexpr int A_TILE = 128 * BK * 2;       // 16 KB
constexpr int B_TILE = NT * BK * 2;        // 8 KB
constexpr int kThreads = 320;              // 10 warps: TMA, MMA, 8 x (converter/metadata + epilogue)
constexpr int kSmemBudget = 196 * 1024;     // pipeline stages; + static VMeta staging + barriers <= 227 KB

struct Bundle {
  int map_a;                 // which A tensor map (0/1)
  int nA; int a_row[4];      // A row offsets (added to the CTA's unit base m0)
  int a_col0;                // A column (k) base
  int nB; int b_col[4];      // B column bases in the arena
  int sum;                   // C = sum of the nB B tiles (child-sum h~)
  int nk;                    // k-blocks
  int nmma; int mma_a[6], mma_b[6], mma_acc[6];   // mma_b: 0..3 B tile, kC = the child-sum tile
};
constexpr int kC = 7;
struct PlanI { int nb; Bundle b[4]; int stages; int stage_bytes; int offB; int offC; };

struct SegT2 { int a_col; int b_col; int k_lo, k_hi; int skip_no_x; };
struct PlanII { int nseg; SegT2 s[4]; int M, Ncols, ldo; int split; size_t split_stride; int stages; };

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~(uintptr_t)1023);
}

// ------------------------------------------------------------------------------------
template <int E, int NACC>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_typeI(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
           const __grid_constant__ CUtensorMap mB, Dev D, PlanI P, int row_lo, int row_hi, int units) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = P.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * P.stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* conv = empty + S;
  uint64_t* done = conv + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int p0 = row_lo + blockIdx.y * NT;
  __shared__ unsigned long long s_tr[6];
  if (D.trace && threadIdx.x == 0) s_tr[0] = gtime();

  __shared__ VMeta s_meta[NT];
  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ || E == EPI_DX) {
    bool act = false;
    if (threadIdx.x < NT) { const int p = p0 + threadIdx.x; act = p < row_hi && row_active<E>(D, p, D.xrow_pos[p]); }
    if (!__syncthreads_or(act)) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); ptx::mbar_init(&conv[s], 128); }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (D.trace && threadIdx.x == 0) s_tr[1] = gtime();

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch(&mA0); ptx::tma_prefetch(&mA1); ptx::tma_prefetch(&mB);
      int step = 0;
      for (int bi = 0; bi < P.nb; ++bi) {
        const Bundle& b = P.b[bi];
        const CUtensorMap* ma = b.map_a ? &mA1 : &mA0;
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * P.stage_bytes;
          ptx::mbar_arrive_expect_tx(&full[s], b.nA * A_TILE + b.nB * B_TILE);
          for (int i = 0; i < b.nA; ++i)
            ptx::tma_load_2d(st + i * A_TILE, ma, b.a_col0 + kb * BK, b.a_row[i] + m0, &full[s]);
          for (int i = 0; i < b.nB; ++i)
            ptx::tma_load_2d(st + P.offB + i * B_TILE, &mB, b.b_col[i] + kb * BK, p0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
      int step = 0;
      for (int bi = 0; bi < P.nb; ++bi) {
        const Bundle& b = P.b[bi];
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&full[s], ph);
          if (b.sum) ptx::mbar_wait(&conv[s], ph);
          ptx::tc_fence_after();
          const uint32_t st = ptx::smem_u32(smem + s * P.stage_bytes);
          for (int m = 0; m < b.nmma; ++m) {
            const uint32_t a = st + b.mma_a[m] * A_TILE;
            const uint32_t bb = b.mma_b[m] == kC ? st + P.offC : st + P.offB + b.mma_b[m] * B_TILE;
            const uint32_t d = tmem + b.mma_acc[m] * NT;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              ptx::mma_bf16(d, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(bb + kk * 32, 16, 1024),
                            idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            }
          }
          ptx::mma_commit(&empty[s]);
        }
      }
      ptx::mma_commit(done);
    }
    __syncwarp();
  } else {
    if (warp < 6) {
      // ---- child-sum converters (h~ = sum_k h_k into the C tile, same swizzled layout) ----
      const int ct = threadIdx.x - 64;          // 0..127
      int step = 0;
      for (int bi = 0; bi < P.nb; ++bi) {
        const Bundle& b = P.b[bi];
        if (!b.sum) { step += b.nk; continue; }
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&full[s], ph);
          uint8_t* st = smem + s * P.stage_bytes;
          for (int c = ct; c < NT * 8; c += 128) {
            const int r = c >> 3, q = c & 7;
            const int off = r * 128 + ((q ^ (r & 7)) << 4);
            float acc[8];
            {
              const uint4 v = *reinterpret_cast<const uint4*>(st + P.offB + off);
              const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] = __bfloat162float(e[i]);
            }
            for (int t = 1; t < b.nB; ++t) {
              const uint4 v = *reinterpret_cast<const uint4*>(st + P.offB + t * B_TILE + off);
              const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(e[i]);
            }
            uint4 o;
            __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
            for (int i = 0; i < 8; ++i) oe[i] = __float2bfloat16_rn(acc[i]);
            *reinterpret_cast<uint4*>(st + P.offC + off) = o;
            const int p = p0 + r;
            if (m0 == 0 && p < row_hi && D.Hs)     // keep h~ for the lazy dU_iou GEMM
              *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(D.Hs) + (size_t)p * D.h + kb * BK + q * 8) = o;
          }
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&conv[s]);
        }
      }
    } else {
      // ---- per-vertex metadata into shared memory while the mainloop runs ----
      const int r = threadIdx.x - 192;
      if (r < NT && p0 + r < row_hi) load_meta(D, p0 + r, epi_needs_children<E>(), s_meta[r]);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    // ---- epilogue: 2 groups of 4 warps, each group 32 of the NT task rows ----
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    if (D.trace && threadIdx.x == 64) s_tr[2] = gtime();
    const int qd = warp & 3;                   // TMEM lane quarter this warp may access
    const int grp = (warp - 2) >> 2;
    const int j = m0 + qd * 32 + lane;
    const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16);
    const UnitC uc = (epi_uses_bias<E>() && j < units) ? load_unit(D, j, epi_is_lstm<E>()) : UnitC{0.f, 0.f, 0.f, 0.f};
    constexpr int CH = epi_needs_children<E>() ? 4 : 8;
    for (int c0 = grp * 32; c0 < grp * 32 + 32; c0 += CH) {
      if (p0 + c0 >= row_hi) break;            // warp-uniform
      float v[NACC][CH];
#pragma unroll
      for (int a = 0; a < NACC; ++a) ptx::tmem_ld<CH>(tq + a * NT + c0, v[a]);
      if (j < units) {
        typename EpiK<E>::In in[CH];
        bool ok[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) {         // all loads of the chunk first ...
          const int r = c0 + i;
          ok[i] = p0 + r < row_hi && row_active<E>(D, p0 + r, s_meta[r].xrow);
          if (ok[i]) EpiK<E>::load(D, j, s_meta[r], in[i]);
        }
#pragma unroll
        for (int i = 0; i < CH; ++i) {         // ... then the math and the stores
          if (!ok[i]) continue;
          float acc[NACC];
#pragma unroll
          for (int a = 0; a < NACC; ++a) acc[a] = v[a][i];
          EpiK<E>::template store<__nv_bfloat16>(D, j, s_meta[c0 + i], acc, in[i], uc);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (D.trace && threadIdx.x == 0) {
    const unsigned long long t = gtime();
    const unsigned long long at = 8 + 8 * atomicAdd(D.trace, 1ull);
    if (at + 8 < (4u << 20) / 8) {
      D.trace[at] = E; D.trace[at + 1] = blockIdx.x + 1000ull * blockIdx.y; D.trace[at + 2] = row_lo;
      D.trace[at + 3] = s_tr[0]; D.trace[at + 4] = s_tr[1]; D.trace[at + 5] = s_tr[2]; D.trace[at + 6] = t;
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
  constexpr int STAGE = 2 * T2_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int* s_count = reinterpret_cast<int*>(tmem_slot + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * 128, z = blockIdx.z;
  // global k-block range of this split
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
  if (warp == 1) ptx::tmem_alloc<128>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch(&mA); ptx::tma_prefetch(&mB);
      int step = 0, g = 0;
      for (int si = 0; si < P.nseg; ++si) {
        const SegT2 sg = P.s[si];
        const int nkb = cdiv(sg.k_hi - sg.k_lo, 64);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          if (g < g_lo || g >= g_hi) continue;
          const int r0 = sg.k_lo + kb * 64;
          if (sg.skip_no_x && !kb_has_x(D, r0)) continue;
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * STAGE;
          ptx::mbar_arrive_expect_tx(&full[s], STAGE);
          ptx::tma_load_2d(st, &mA, sg.a_col + m0, r0, &full[s]);
          ptx::tma_load_2d(st + T2_TILE / 2, &mA, sg.a_col + m0 + 64, r0, &full[s]);
          ptx::tma_load_2d(st + T2_TILE, &mB, sg.b_col + n0, r0, &full[s]);
          ptx::tma_load_2d(st + T2_TILE + T2_TILE / 2, &mB, sg.b_col + n0 + 64, r0, &full[s]);
          ++step;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(128, 128, 1, 1);
      int step = 0, g = 0;
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
          const uint32_t a = ptx::smem_u32(smem + s * STAGE);
          const uint32_t b = a + T2_TILE;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_bf16(tmem, ptx::sdesc_sw128(a + kk * 2048, 8192, 1024), ptx::sdesc_sw128(b + kk * 2048, 8192, 1024),
                          idesc, (step > 0 || kk > 0) ? 1u : 0u);
          ptx::mma_commit(&empty[s]);
          ++step;
        }
      }
      *s_count = step;
      ptx::mma_commit(done);
    }
    __syncwarp();
  } else if (warp < 6) {
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
      if (m < P.M) {
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c + i;
          if (n < P.Ncols) o[(size_t)m * P.ldo + n] = any ? v[i] : 0.f;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<128>(tmem);
  }
}


// ------------------------------------------------------------------------------------
// Gate-split cluster level kernel.  A cluster of 4 CTAs covers one 128-unit block of one
// 64-row task tile; rank r streams only its gate's weights (forward: U_i / U_o / U_u / U_f;
// backward and dX: the K columns of gate r), so each CTA pulls ~1/4 of the weights of the
// monolithic kernel.  After the mainloop every CTA stages its accumulators in its own shared
// memory, the cluster synchronises, and rank r runs the fused cell epilogue for task columns
// [16r, 16r+16), reading the other ranks' accumulators through distributed shared memory.
constexpr int kCluster = 4;
constexpr int kOwn = NT / kCluster;   // task columns per CTA in the epilogue

struct RankPlan { int nb; Bundle b[3]; int nacc; int stages; int stage_bytes; int offB; int offC; };
struct PlanGS { RankPlan r[kCluster]; int comb[8][kCluster]; int bar_off; };

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
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

template <int E, int NACC>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gs(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
        const __grid_constant__ CUtensorMap mB, Dev D, PlanGS P, int row_lo, int row_hi, int units) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const uint32_t rank = cluster_rank();
  const RankPlan& R = P.r[rank];
  const int S = R.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bar_off);
  uint64_t* empty = full + 6;
  uint64_t* conv = empty + 6;
  uint64_t* done = conv + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* xs = reinterpret_cast<float*>(smem);                    // [nacc][NT][128] after the mainloop
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (blockIdx.x / kCluster) * 128;
  const int p0 = row_lo + blockIdx.y * NT;
  __shared__ VMeta s_meta[kOwn];

  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ || E == EPI_DX) {
    bool act = false;                                            // uniform across the cluster
    if (threadIdx.x < NT) { const int p = p0 + threadIdx.x; act = p < row_hi && row_active<E>(D, p, D.xrow_pos[p]); }
    if (!__syncthreads_or(act)) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); ptx::mbar_init(&conv[s], 128); }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<256>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::tma_prefetch(&mA0); ptx::tma_prefetch(&mA1); ptx::tma_prefetch(&mB);
      int step = 0;
      for (int bi = 0; bi < R.nb; ++bi) {
        const Bundle& b = R.b[bi];
        const CUtensorMap* ma = b.map_a ? &mA1 : &mA0;
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * R.stage_bytes;
          ptx::mbar_arrive_expect_tx(&full[s], b.nA * A_TILE + b.nB * B_TILE);
          for (int i = 0; i < b.nA; ++i)
            ptx::tma_load_2d(st + i * A_TILE, ma, b.a_col0 + kb * BK, b.a_row[i] + m0, &full[s]);
          for (int i = 0; i < b.nB; ++i)
            ptx::tma_load_2d(st + R.offB + i * B_TILE, &mB, b.b_col[i] + kb * BK, p0, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
      uint32_t written = 0;                                      // accumulators already initialised
      int step = 0;
      for (int bi = 0; bi < R.nb; ++bi) {
        const Bundle& b = R.b[bi];
        for (int kb = 0; kb < b.nk; ++kb, ++step) {
          const int s = step % S;
          const uint32_t ph = (step / S) & 1;
          ptx::mbar_wait(&full[s], ph);
          if (b.sum) ptx::mbar_wait(&conv[s], ph);
          ptx::tc_fence_after();
          const uint32_t st = ptx::smem_u32(smem + s * R.stage_bytes);
          for (int m = 0; m < b.nmma; ++m) {
            const uint32_t a = st + b.mma_a[m] * A_TILE;
            const uint32_t bb = b.mma_b[m] == kC ? st + R.offC : st + R.offB + b.mma_b[m] * B_TILE;
            const int acc = b.mma_acc[m];
            const uint32_t d = tmem + acc * NT;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              ptx::mma_bf16(d, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(bb + kk * 32, 16, 1024),
                            idesc, ((written >> acc) & 1u) | (kk > 0 ? 1u : 0u));
            }
            written |= 1u << acc;
          }
          ptx::mma_commit(&empty[s]);
        }
      }
      ptx::mma_commit(done);
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---- child-sum converters ----
    const int ct = threadIdx.x - 64;
    int step = 0;
    for (int bi = 0; bi < R.nb; ++bi) {
      const Bundle& b = R.b[bi];
      if (!b.sum) { step += b.nk; continue; }
      for (int kb = 0; kb < b.nk; ++kb, ++step) {
        const int s = step % S;
        const uint32_t ph = (step / S) & 1;
        ptx::mbar_wait(&full[s], ph);
        uint8_t* st = smem + s * R.stage_bytes;
        for (int c = ct; c < NT * 8; c += 128) {
          const int r = c >> 3, q = c & 7;
          const int off = r * 128 + ((q ^ (r & 7)) << 4);
          float acc[8];
          {
            const uint4 v = *reinterpret_cast<const uint4*>(st + R.offB + off);
            const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __bfloat162float(e[i]);
          }
          for (int t = 1; t < b.nB; ++t) {
            const uint4 v = *reinterpret_cast<const uint4*>(st + R.offB + t * B_TILE + off);
            const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(e[i]);
          }
          uint4 o;
          __nv_bfloat16* oe = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
          for (int i = 0; i < 8; ++i) oe[i] = __float2bfloat16_rn(acc[i]);
          *reinterpret_cast<uint4*>(st + R.offC + off) = o;
          const int p = p0 + r;
          if (m0 == 0 && rank == 0 && p < row_hi && D.Hs)        // keep h~ for the lazy dU_iou GEMM
            *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(D.Hs) + (size_t)p * D.h + kb * BK + q * 8) = o;
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&conv[s]);
      }
    }
  } else {
    // ---- metadata of this CTA's epilogue columns ----
    const int r = threadIdx.x - 192;
    const int p = p0 + (int)rank * kOwn + r;
    if (r < kOwn && p < row_hi) load_meta(D, p, epi_needs_children<E>(), s_meta[r]);
  }
  // ---- stage own accumulators in shared memory ----
  const int qd = warp & 3;
  if (warp >= 2) {
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    const int grp = (warp - 2) >> 2;
    const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16);
    for (int a = 0; a < R.nacc; ++a) {
      for (int c0 = grp * 32; c0 < grp * 32 + 32; c0 += 8) {
        float v[8];
        ptx::tmem_ld<8>(tq + a * NT + c0, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) xs[((size_t)a * NT + c0 + i) * 128 + qd * 32 + lane] = v[i];
      }
    }
  }
  ptx::tc_fence_before();
  cluster_sync_all();
  // ---- fused epilogue over this CTA's kOwn columns (two groups of 8) ----
  if (warp >= 2) {
    const int grp = (warp - 2) >> 2;
    const int j = m0 + qd * 32 + lane;
    const UnitC uc = (epi_uses_bias<E>() && j < units) ? load_unit(D, j, epi_is_lstm<E>()) : UnitC{0.f, 0.f, 0.f, 0.f};
    const uint32_t xs_base = ptx::smem_u32(xs) + (uint32_t)(qd * 32 + lane) * 4u;
    constexpr int CH = epi_needs_children<E>() ? 2 : 8;        // vertices whose loads are batched
#pragma unroll 1
    for (int c0 = 0; c0 < kOwn / 2; c0 += CH) {
      float acc[CH][NACC];
      typename EpiK<E>::In in[CH];
      bool ok[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int r = grp * (kOwn / 2) + c0 + i;               // own-column index
        const int c = (int)rank * kOwn + r;                    // task column in the tile
        const int p = p0 + c;
        ok[i] = j < units && p < row_hi && row_active<E>(D, p, s_meta[r].xrow);
        if (!ok[i]) continue;
#pragma unroll
        for (int e = 0; e < NACC; ++e) {
          float sum = 0.f;
#pragma unroll
          for (int q = 0; q < kCluster; ++q) {
            const int ai = P.comb[e][q];
            if (ai >= 0) sum += ld_dsmem(mapa_rank(xs_base + (uint32_t)((ai * NT + c) * 128) * 4u, q));
          }
          acc[i][e] = sum;
        }
        EpiK<E>::load(D, j, s_meta[r], in[i]);
      }
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (ok[i]) EpiK<E>::template store<__nv_bfloat16>(D, j, s_meta[grp * (kOwn / 2) + c0 + i], acc[i], in[i], uc);
    }
  }
  cluster_sync_all();                                          // remote reads done before smem is released
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
  CUtensorMap M_dz, M_hs, M_hk, M_xp;
  bool use_simt = false;
  bool mono = false;            // CAVS_TC_MONO=1: one CTA per 128-unit block (A/B checks)
};

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

cavs_status tc_init(const Dev& D, int max_vertices, TcState** out, std::string* err) {
  TcState* t = new TcState();
  const char* env = std::getenv("CAVS_BF16_SIMT");
  t->use_simt = env && env[0] == '1';
  const char* mono = std::getenv("CAVS_TC_MONO");
  t->mono = mono && mono[0] == '1';
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
  bool ok = true;
  if (lstm) {
    ok &= encode(&t->A[0], D.Wa, h, 4 * h, h, BK, 128);          // U4   [4h x h]
    ok &= encode(&t->A[1], D.Wb, d, 4 * h, d, BK, 128);          // W4   [4h x d]
    ok &= encode(&t->A[2], D.Wc, 3 * h, h, 3 * h, BK, 128);      // UTiou[h x 3h]
    ok &= encode(&t->A[3], D.Wd, h, h, h, BK, 128);              // UTf  [h x h]
    ok &= encode(&t->A[4], D.We, G * h, d, G * h, BK, 128);      // WT   [d x G h]
  } else {
    ok &= encode(&t->A[0], D.Wa, 2 * h, h, 2 * h, BK, 128);      // Wc   [h x 2h]
    ok &= encode(&t->A[1], D.Wb, d, h, d, BK, 128);              // Wx   [h x d]
    ok &= encode(&t->A[2], D.Wc, h, 2 * h, h, BK, 128);          // WcT  [2h x h]
    t->A[3] = t->A[2];
    ok &= encode(&t->A[4], D.We, h, d, h, BK, 128);              // WxT  [d x h]
  }
  ok &= encode(&t->B_hk, D.Hk, N * h, Vp, N * h, BK, NT);
  ok &= encode(&t->B_xp, D.Xp, d, Vp, d, BK, NT);
  ok &= encode(&t->B_dz, D.dZ, G * h, Vp, G * h, BK, NT);
  ok &= encode(&t->M_dz, D.dZ, G * h, Vp, G * h, 64, 64);
  ok &= encode(&t->M_hk, D.Hk, N * h, Vp, N * h, 64, 64);
  ok &= encode(&t->M_xp, D.Xp, d, Vp, d, 64, 64);
  if (D.Hs) ok &= encode(&t->M_hs, D.Hs, h, Vp, h, 64, 64);
  if (!ok) {
    *err = "cuTensorMapEncodeTiled failed";
    delete t;
    return CAVS_E_CUDA;
  }
  *out = t;
  return CAVS_OK;
}

void tc_destroy(TcState* tc) { delete tc; }

static int finalize(PlanI& P) {
  int maxA = 0, maxB = 0, sum = 0;
  for (int i = 0; i < P.nb; ++i) {
    maxA = std::max(maxA, P.b[i].nA);
    maxB = std::max(maxB, P.b[i].nB);
    sum |= P.b[i].sum;
  }
  P.offB = maxA * A_TILE;
  P.offC = P.offB + maxB * B_TILE;
  P.stage_bytes = P.offC + (sum ? B_TILE : 0);
  P.stages = std::max(1, std::min(6, kSmemBudget / P.stage_bytes));
  return P.stages * P.stage_bytes + 1024 + 3 * 8 * P.stages + 64;
}

template <int E, int NACC>
static void launch_I(const TcState* t, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                     const Dev& D, PlanI P, int row_lo, int row_hi, int units, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  const int smem = finalize(P);
  static int attr_set = 0;                     // dynamic + static smem must stay <= 227 KB
  if (smem > attr_set) {
    cudaFuncSetAttribute(k_tc_typeI<E, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = smem;
  }
  dim3 grid(cdiv(units, 128), cdiv(row_hi - row_lo, NT));
  k_tc_typeI<E, NACC><<<grid, kThreads, smem, s>>>(a0, a1, b, D, P, row_lo, row_hi, units);
}

static Bundle one(int map_a, int a_row, int a_col0, int b_col, int nk, int acc) {
  Bundle b{};
  b.map_a = map_a; b.nA = 1; b.a_row[0] = a_row; b.a_col0 = a_col0;
  b.nB = 1; b.b_col[0] = b_col; b.sum = 0; b.nk = nk;
  b.nmma = 1; b.mma_a[0] = 0; b.mma_b[0] = 0; b.mma_acc[0] = acc;
  return b;
}



// ---- gate-split plans ------------------------------------------------------------------
static Bundle bundle(int map_a, int a_row, int a_col0, int nB, const int* b_cols, int sum, int nk) {
  Bundle b{};
  b.map_a = map_a; b.nA = 1; b.a_row[0] = a_row; b.a_col0 = a_col0;
  b.nB = nB; for (int i = 0; i < nB; ++i) b.b_col[i] = b_cols[i];
  b.sum = sum; b.nk = nk;
  return b;
}

static int gs_finalize(PlanGS& P) {
  int pipe = 0, xs = 0;
  for (int r = 0; r < kCluster; ++r) {
    RankPlan& R = P.r[r];
    int maxB = 0, sum = 0;
    for (int i = 0; i < R.nb; ++i) { maxB = std::max(maxB, R.b[i].nB); sum |= R.b[i].sum; }
    R.offB = A_TILE;
    R.offC = R.offB + maxB * B_TILE;
    R.stage_bytes = R.offC + (sum ? B_TILE : 0);
    R.stages = std::max(1, std::min(6, kSmemBudget / R.stage_bytes));
    pipe = std::max(pipe, R.stages * R.stage_bytes);
    xs = std::max(xs, R.nacc * NT * 128 * 4);
  }
  P.bar_off = (std::max(pipe, xs) + 1023) & ~1023;
  return 1024 + P.bar_off + 3 * 6 * 8 + 16 + 64;
}

// K range [0, nkb) k-blocks split over the cluster ranks (contiguous, balanced).
static void ksplit(int nkb, int r, int* kb0, int* nk) {
  const int q = nkb / kCluster, rem = nkb % kCluster;
  *kb0 = r * q + std::min(r, rem);
  *nk = q + (r < rem ? 1 : 0);
}

// all ranks: one bundle over their K share of (A rows a_row, A cols a_col, B cols b_col) -> acc
static void gs_add_ksplit(PlanGS& P, int map_a, int a_row, int a_col, int b_col, int K, int acc) {
  const int nkb = K / BK;
  for (int r = 0; r < kCluster; ++r) {
    int kb0, nk;
    ksplit(nkb, r, &kb0, &nk);
    RankPlan& R = P.r[r];
    if (nk == 0) continue;
    const int bc = b_col + kb0 * BK;
    Bundle b = bundle(map_a, a_row, a_col + kb0 * BK, 1, &bc, 0, nk);
    b.nmma = 1; b.mma_a[0] = 0; b.mma_b[0] = 0; b.mma_acc[0] = R.nacc;
    R.b[R.nb++] = b;
    P.comb[acc][r] = R.nacc;
    R.nacc++;
  }
}

static PlanGS gs_empty() {
  PlanGS P{};
  for (int e = 0; e < 8; ++e) for (int r = 0; r < kCluster; ++r) P.comb[e][r] = -1;
  return P;
}

// Tree-LSTM forward task: rank g < 3 -> gate g over h~; rank 3 -> U_f over every child slot.
static PlanGS gs_lstm_fwd(int h, int N) {
  PlanGS P = gs_empty();
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = k * h;
  for (int g = 0; g < 3; ++g) {
    RankPlan& R = P.r[g];
    Bundle b = bundle(0, g * h, 0, N, cols, N >= 2, h / BK);
    b.nmma = 1; b.mma_a[0] = 0; b.mma_b[0] = N >= 2 ? kC : 0; b.mma_acc[0] = 0;
    R.b[0] = b; R.nb = 1; R.nacc = 1;
    P.comb[g][g] = 0;
  }
  RankPlan& R = P.r[3];
  Bundle b = bundle(0, 3 * h, 0, N, cols, 0, h / BK);
  b.nmma = N;
  for (int k = 0; k < N; ++k) { b.mma_a[k] = 0; b.mma_b[k] = k; b.mma_acc[k] = k; P.comb[3 + k][3] = k; }
  R.b[0] = b; R.nb = 1; R.nacc = N;
  return P;
}

// Tree-LSTM eager pull projection: rank g -> gate g of W4 over Xp.
static PlanGS gs_lstm_xproj(int h, int d) {
  PlanGS P = gs_empty();
  const int zero = 0;
  for (int g = 0; g < 4; ++g) {
    RankPlan& R = P.r[g];
    Bundle b = bundle(0, g * h, 0, 1, &zero, 0, d / BK);
    b.nmma = 1; b.mma_a[0] = 0; b.mma_b[0] = 0; b.mma_acc[0] = 0;
    R.b[0] = b; R.nb = 1; R.nacc = 1;
    P.comb[g][g] = 0;
  }
  return P;
}

// Tree-LSTM backward task: rank g < 3 -> U_g^T dz_g (K = gate g); rank 3 -> U_f^T dz_fk per slot.
static PlanGS gs_lstm_bwd(int h, int N) {
  PlanGS P = gs_empty();
  for (int g = 0; g < 3; ++g) {
    RankPlan& R = P.r[g];
    const int bc = g * h;
    Bundle b = bundle(0, 0, g * h, 1, &bc, 0, h / BK);
    b.nmma = 1; b.mma_a[0] = 0; b.mma_b[0] = 0; b.mma_acc[0] = 0;
    R.b[0] = b; R.nb = 1; R.nacc = 1;
    P.comb[0][g] = 0;
  }
  RankPlan& R = P.r[3];
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = (3 + k) * h;
  Bundle b = bundle(1, 0, 0, N, cols, 0, h / BK);
  b.nmma = N;
  for (int k = 0; k < N; ++k) { b.mma_a[k] = 0; b.mma_b[k] = k; b.mma_acc[k] = k; P.comb[1 + k][3] = k; }
  R.b[0] = b; R.nb = 1; R.nacc = N;
  return P;
}

// Tree-LSTM dX: rank g < 3 -> W_g^T dz_g; rank 3 -> W_f^T sum_k dz_fk (one acc).
static PlanGS gs_lstm_dx(int h, int N) {
  PlanGS P = gs_empty();
  for (int g = 0; g < 3; ++g) {
    RankPlan& R = P.r[g];
    const int bc = g * h;
    Bundle b = bundle(0, 0, g * h, 1, &bc, 0, h / BK);
    b.nmma = 1; b.mma_a[0] = 0; b.mma_b[0] = 0; b.mma_acc[0] = 0;
    R.b[0] = b; R.nb = 1; R.nacc = 1;
    P.comb[0][g] = 0;
  }
  RankPlan& R = P.r[3];
  int cols[4];
  for (int k = 0; k < N; ++k) cols[k] = (3 + k) * h;
  Bundle b = bundle(0, 0, 3 * h, N, cols, 0, h / BK);
  b.nmma = N;
  for (int k = 0; k < N; ++k) { b.mma_a[k] = 0; b.mma_b[k] = k; b.mma_acc[k] = 0; }
  R.b[0] = b; R.nb = 1; R.nacc = 1;
  P.comb[0][3] = 0;
  return P;
}

template <int E, int NACC>
static void launch_gs(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b, const Dev& D, PlanGS P,
                      int row_lo, int row_hi, int units, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  const int smem = gs_finalize(P);
  static int attr_set = 0;
  if (smem > attr_set) {
    cudaFuncSetAttribute(k_tc_gs<E, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCluster * cdiv(units, 128), cdiv(row_hi - row_lo, NT), 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_tc_gs<E, NACC>, a0, a1, b, D, P, row_lo, row_hi, units);
}

void tc_forward(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, Prof& P) {
  const int skmax = skinny_max(D);
  if (t->use_simt) { simt_forward<__nv_bfloat16>(D, lp, s, P); return; }
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    // eager pull projection + level 0: A = W4 (gates i,o,u,f), B = Xp
    PlanI X{};
    X.nb = 1;
    Bundle& b = X.b[0];
    b.map_a = 0; b.nA = 4; for (int g = 0; g < 4; ++g) b.a_row[g] = g * h; b.a_col0 = 0;
    b.nB = 1; b.b_col[0] = 0; b.sum = 0; b.nk = d / BK;
    b.nmma = 4; for (int g = 0; g < 4; ++g) { b.mma_a[g] = g; b.mma_b[g] = 0; b.mma_acc[g] = g; }
    if (t->mono) launch_I<EPI_LSTM_XPROJ, 4>(t, t->A[1], t->A[1], t->B_xp, D, X, 0, D.V, h, s);
    else launch_gs<EPI_LSTM_XPROJ, 4>(t->A[1], t->A[1], t->B_xp, D, gs_lstm_xproj(h, d), 0, D.V, h, s);
    P.count(1);
    P.mark(CAVS_PH_FWD_LEVELS, s);
    // levels t >= 1: A = U4, B = child slots of the task's rows; h~ formed in smem
    PlanI F{};
    F.nb = 1;
    Bundle& f = F.b[0];
    f.map_a = 0; f.nA = 4; for (int g = 0; g < 4; ++g) f.a_row[g] = g * h; f.a_col0 = 0;
    f.nB = N; for (int k = 0; k < N; ++k) f.b_col[k] = k * h;
    f.sum = N >= 2; f.nk = h / BK;
    f.nmma = 3 + N;
    for (int g = 0; g < 3; ++g) { f.mma_a[g] = g; f.mma_b[g] = N >= 2 ? kC : 0; f.mma_acc[g] = g; }
    for (int k = 0; k < N; ++k) { f.mma_a[3 + k] = 3; f.mma_b[3 + k] = k; f.mma_acc[3 + k] = 3 + k; }
    const SegListI Fs = fwd_segments(D);
    const PlanGS G = gs_lstm_fwd(h, N);
    for (int tt = 1; tt < T; ++tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_FWD, Fs, lp[tt], lp[tt + 1], h, s);
      else if (!t->mono) {
        if (N == 1) launch_gs<EPI_LSTM_FWD, 4>(t->A[0], t->A[0], t->B_hk, D, G, lp[tt], lp[tt + 1], h, s);
        else if (N == 2) launch_gs<EPI_LSTM_FWD, 5>(t->A[0], t->A[0], t->B_hk, D, G, lp[tt], lp[tt + 1], h, s);
        else if (N == 3) launch_gs<EPI_LSTM_FWD, 6>(t->A[0], t->A[0], t->B_hk, D, G, lp[tt], lp[tt + 1], h, s);
        else launch_gs<EPI_LSTM_FWD, 7>(t->A[0], t->A[0], t->B_hk, D, G, lp[tt], lp[tt + 1], h, s);
      } else if (N == 1) launch_I<EPI_LSTM_FWD, 4>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      else if (N == 2) launch_I<EPI_LSTM_FWD, 5>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      else if (N == 3) launch_I<EPI_LSTM_FWD, 6>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      else launch_I<EPI_LSTM_FWD, 7>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      P.count(1);
    }
  } else {
    PlanI X{};
    X.nb = 1;
    X.b[0] = one(0, 0, 0, 0, d / BK, 0);
    if (t->mono) launch_I<EPI_FC_XPROJ, 1>(t, t->A[1], t->A[1], t->B_xp, D, X, 0, D.V, h, s);
    else {
      PlanGS G = gs_empty();
      gs_add_ksplit(G, 0, 0, 0, 0, d, 0);
      launch_gs<EPI_FC_XPROJ, 1>(t->A[1], t->A[1], t->B_xp, D, G, 0, D.V, h, s);
    }
    P.count(1);
    P.mark(CAVS_PH_FWD_LEVELS, s);
    PlanI F{};
    F.nb = 1;
    F.b[0] = one(0, 0, 0, 0, 2 * h / BK, 0);
    const SegListI Fs = fwd_segments(D);
    PlanGS G = gs_empty();
    gs_add_ksplit(G, 0, 0, 0, 0, 2 * h, 0);
    for (int tt = 1; tt < T; ++tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_FWD, Fs, lp[tt], lp[tt + 1], h, s);
      else if (!t->mono) launch_gs<EPI_FC_FWD, 1>(t->A[0], t->A[0], t->B_hk, D, G, lp[tt], lp[tt + 1], h, s);
      else launch_I<EPI_FC_FWD, 1>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      P.count(1);
    }
  }
}

static int launch_II(const CUtensorMap& a, const CUtensorMap& b, const Dev& D, PlanII P, float* out,
                     cudaStream_t s) {
  int nkb = 0;
  for (int i = 0; i < P.nseg; ++i) nkb += cdiv(P.s[i].k_hi - P.s[i].k_lo, 64);
  const int tiles = cdiv(P.M, 128) * cdiv(P.Ncols, 128);
  P.split = std::max(1, std::min(std::min(kSplitMax, 148 / std::max(1, tiles)), std::max(1, nkb / 4)));
  P.stages = 6;
  const int smem = P.stages * 2 * T2_TILE + 1024 + 2 * 8 * P.stages + 64;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(k_tc_typeII, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = true;
  }
  dim3 grid(cdiv(P.M, 128), cdiv(P.Ncols, 128), P.split);
  k_tc_typeII<<<grid, kThreads, smem, s>>>(a, b, D, P, out);
  return P.split;
}

void tc_backward(Dev& D, TcState* t, const std::vector<int>& lp, cudaStream_t s, int* split, Prof& P) {
  const int skmax = skinny_max(D);
  split[0] = split[1] = split[2] = 1;
  if (t->use_simt) { simt_backward<__nv_bfloat16>(D, lp, s, P); return; }
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int G = lstm ? 3 + N : 1;
  // rows past V of dZ are read by the lazy GEMMs' last k-block: keep them zero
  cudaMemsetAsync(reinterpret_cast<__nv_bfloat16*>(D.dZ) + (size_t)D.V * G * h, 0, (size_t)64 * G * h * 2, s);
  if (lstm) {
    PlanI B{};
    B.nb = 1 + N;
    B.b[0] = one(0, 0, 0, 0, 3 * h / BK, 0);                          // UTiou x dZ_iou
    for (int k = 0; k < N; ++k) B.b[1 + k] = one(1, 0, 0, (3 + k) * h, h / BK, 1 + k);   // UTf x dZ_fk
    const SegListI Bs = bwd_segments(D);
    const PlanGS G = gs_lstm_bwd(h, N);
    for (int tt = T - 1; tt >= 1; --tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_BWD, Bs, lp[tt], lp[tt + 1], h, s);
      else if (!t->mono) {
        if (N == 1) launch_gs<EPI_LSTM_BWD, 2>(t->A[2], t->A[3], t->B_dz, D, G, lp[tt], lp[tt + 1], h, s);
        else if (N == 2) launch_gs<EPI_LSTM_BWD, 3>(t->A[2], t->A[3], t->B_dz, D, G, lp[tt], lp[tt + 1], h, s);
        else if (N == 3) launch_gs<EPI_LSTM_BWD, 4>(t->A[2], t->A[3], t->B_dz, D, G, lp[tt], lp[tt + 1], h, s);
        else launch_gs<EPI_LSTM_BWD, 5>(t->A[2], t->A[3], t->B_dz, D, G, lp[tt], lp[tt + 1], h, s);
      } else if (N == 1) launch_I<EPI_LSTM_BWD, 2>(t, t->A[2], t->A[3], t->B_dz, D, B, lp[tt], lp[tt + 1], h, s);
      else if (N == 2) launch_I<EPI_LSTM_BWD, 3>(t, t->A[2], t->A[3], t->B_dz, D, B, lp[tt], lp[tt + 1], h, s);
      else if (N == 3) launch_I<EPI_LSTM_BWD, 4>(t, t->A[2], t->A[3], t->B_dz, D, B, lp[tt], lp[tt + 1], h, s);
      else launch_I<EPI_LSTM_BWD, 5>(t, t->A[2], t->A[3], t->B_dz, D, B, lp[tt], lp[tt + 1], h, s);
      P.count(1);
    }
  } else {
    PlanI B{};
    B.nb = 2;
    for (int k = 0; k < 2; ++k) B.b[k] = one(0, k * h, 0, 0, h / BK, k);   // WcT rows k*h x dZ
    const SegListI Bs = bwd_segments(D);
    PlanGS G = gs_empty();
    for (int k = 0; k < 2; ++k) gs_add_ksplit(G, 0, k * h, 0, 0, h, k);
    for (int tt = T - 1; tt >= 1; --tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_BWD, Bs, lp[tt], lp[tt + 1], h, s);
      else if (!t->mono) launch_gs<EPI_FC_BWD, 2>(t->A[2], t->A[2], t->B_dz, D, G, lp[tt], lp[tt + 1], h, s);
      else launch_I<EPI_FC_BWD, 2>(t, t->A[2], t->A[2], t->B_dz, D, B, lp[tt], lp[tt + 1], h, s);
      P.count(1);
    }
  }
  P.mark(CAVS_PH_LAZY, s);
  // ---- lazy batching of the parameter gradients ----
  const size_t su4 = lstm ? (size_t)3 * h * h : (size_t)2 * h * h;
  const size_t suf = lstm ? (size_t)h * h : 0;
  const size_t sw = (size_t)G * h * d;
  float* u4 = D.lazy;
  float* uf = u4 + kSplitMax * su4;
  float* w = uf + kSplitMax * suf;
  const int lp1 = D.lp1, V = D.V;
  if (lstm) {
    PlanII A{};
    A.nseg = 1;
    A.s[0] = SegT2{0, 0, lp1, V, 0};
    A.M = 3 * h; A.Ncols = h; A.ldo = h; A.split_stride = su4;
    if (lp1 < V) { split[0] = launch_II(t->M_dz, N >= 2 ? t->M_hs : t->M_hk, D, A, u4, s); P.count(1); }
    else cudaMemsetAsync(u4, 0, sizeof(float) * su4, s);
    PlanII Bf{};
    Bf.nseg = N;
    for (int k = 0; k < N; ++k) Bf.s[k] = SegT2{(3 + k) * h, k * h, lp1, V, 0};
    Bf.M = h; Bf.Ncols = h; Bf.ldo = h; Bf.split_stride = suf;
    if (lp1 < V) { split[1] = launch_II(t->M_dz, t->M_hk, D, Bf, uf, s); P.count(1); }
    else cudaMemsetAsync(uf, 0, sizeof(float) * suf, s);
    PlanII Cw{};
    Cw.nseg = 1;
    Cw.s[0] = SegT2{0, 0, 0, V, 1};
    Cw.M = G * h; Cw.Ncols = d; Cw.ldo = d; Cw.split_stride = sw;
    split[2] = launch_II(t->M_dz, t->M_xp, D, Cw, w, s); P.count(1);
    P.mark(CAVS_PH_DX, s);
    if (D.dx) {
      PlanI X{};
      X.nb = 1;
      X.b[0] = one(0, 0, 0, 0, G * h / BK, 0);
      if (t->mono) launch_I<EPI_DX, 1>(t, t->A[4], t->A[4], t->B_dz, D, X, 0, V, d, s);
      else launch_gs<EPI_DX, 1>(t->A[4], t->A[4], t->B_dz, D, gs_lstm_dx(h, N), 0, V, d, s);
      P.count(1);
    }
  } else {
    float* wc = u4;
    float* wx = w;
    PlanII A{};
    A.nseg = 1;
    A.s[0] = SegT2{0, 0, lp1, V, 0};
    A.M = h; A.Ncols = 2 * h; A.ldo = 2 * h; A.split_stride = su4;
    if (lp1 < V) { split[0] = launch_II(t->M_dz, t->M_hk, D, A, wc, s); P.count(1); }
    else cudaMemsetAsync(wc, 0, sizeof(float) * su4, s);
    PlanII Cw{};
    Cw.nseg = 1;
    Cw.s[0] = SegT2{0, 0, 0, V, 1};
    Cw.M = h; Cw.Ncols = d; Cw.ldo = d; Cw.split_stride = (size_t)h * d;
    split[2] = launch_II(t->M_dz, t->M_xp, D, Cw, wx, s); P.count(1);
    P.mark(CAVS_PH_DX, s);
    if (D.dx) {
      PlanI X{};
      X.nb = 1;
      X.b[0] = one(0, 0, 0, 0, h / BK, 0);
      if (t->mono) launch_I<EPI_DX, 1>(t, t->A[4], t->A[4], t->B_dz, D, X, 0, V, d, s);
      else {
        PlanGS Gx = gs_empty();
        gs_add_ksplit(Gx, 0, 0, 0, 0, h, 0);
        launch_gs<EPI_DX, 1>(t->A[4], t->A[4], t->B_dz, D, Gx, 0, V, d, s);
      }
      P.count(1);
    }
  }
}

}  // namespace cavs
