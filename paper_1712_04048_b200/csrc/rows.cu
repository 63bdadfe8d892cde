// rows.cu — BF16 mode: row-tiled tcgen05 level GEMMs for LARGE tasks when the weights of F do
// not fit the persistent weight-stationary kernel (h > 512; Alg. 1 FORWARD/BACKWARD
// task loop P:L362-380, one launch per task V_t, fused cell epilogue as in Fig. 5).
//
// A large task (M_t rows) is a plain dense contraction: Z[rows, units] = A[rows, K] W[units, K]^T
// with A = the task's contiguous rows of the gather arena Hk (forward) or of dZ (backward),
// K-major, and W = F's weights, K-major.  Unlike the per-task swap-AB kernel (tc.cu: 128 weight
// rows x 64 task rows, 45 FLOP/B of operand traffic) the tile here is 128 task rows x 256
// weight rows (87 FLOP/B), so the k-loop is not bound by L2 bandwidth.  The kernel is
// persistent over the task's (row tile, unit tile) pairs; two TMEM accumulator buffers where
// they fit, so the cell epilogue of one tile overlaps the next tile's k-loop.
//
// MMA segments (host plan): segment s multiplies A columns [a_col, a_col + 64 nkb) with the B
// boxes of weight rows {b_row0[g] + u0} into TMEM columns [acc_col, acc_col + n):
//   Tree-FC fwd : 1 segment,  A = Hk [h_l | h_r] (K = 2h), B = W_c rows u0..u0+255   -> z
//   Tree-FC bwd : 1 segment,  A = dZ (K = h), B = W_c^T rows {u0, h + u0} (2 x 128) -> dh_l, dh_r
//   Tree-LSTM fwd: N segments, A = Hk slot k (K = h), B = U rows {i, o, u, f} x 64 units
//                  -> block k = (U_iou h_k, U_f h_k); the epilogue sums the iou parts over k
//                  (U h~ = sum_k U h_k, linearity, Z11)
//   Tree-LSTM bwd: 1 + N segments, A = dZ_iou (K = 3h) x U_iou^T rows u0..u0+127 -> dh~,
//                  A = dZ_fk (K = h) x U_f^T rows -> U_f^T dz_fk
// Epilogue: thread = task row (TMEM lane) x half of the tile's units; per 4-unit quad the
// accumulators are read straight from TMEM and the cell (cells.cuh EpiK) runs in registers.
//   warp 0: TMA producer, warp 1: TMEM allocator + MMA issuer, warps 2-9: epilogue.
// CTA pairs (CG = 2, opt-in CAVS_ROWS_PAIR=1): a cluster of two CTAs on one TPC runs each tile as ONE
// tcgen05.mma.cta_group::2 of M = 256 task rows (128 per CTA) x N = n weight rows, issued by the
// rank-0 CTA; each CTA stages its own 128 A rows and HALF of the B rows (n/2), so a stage is
// 16 KB + n/2 x 128 B instead of 16 KB + n x 128 B: half the weight traffic per SM and 6-8
// pipeline stages instead of 4.  Both CTAs' TMA complete on the leader's full barrier; the
// leader's commits multicast to both CTAs' empty / accumulator-full barriers; both epilogues
// drain their own TMEM and arrive on the leader's accumulator-empty barrier.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "cells.cuh"
#include "ptx.cuh"
#include "rows.h"

namespace cavs {

constexpr int kRThreads = 320;
constexpr int kRSMax = 8;              // pipeline stages (plan: as many as fit shared memory)
constexpr int kRA = 128 * 128;         // A stage: 128 rows x 64 k (bf16) = 16 KB
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;   // shared::cluster address of the pair's rank-0 CTA

struct RSeg { int a_col, bmap, nbox, box_rows, b_row0[4], nkb, acc_col; };
struct RPlan {
  int nseg;
  RSeg seg[5];
  int UG;          // units per tile
  int n;           // MMA N (nbox * box_rows), the same for every segment
  int stage;       // bytes per stage (per CTA)
  int S;           // pipeline stages
  int acc_cols;    // TMEM columns per accumulator buffer
  int nbuf;        // accumulator buffers (1 or 2)
  int lo, hi;      // task rows
  int nut, ntiles; // unit tiles, tiles (of 128 CG task rows)
  int dsm;         // split-K through DSMEM: the ks shares of a tile form a cluster and exchange partials in
                   // shared memory (when a partial fits the pipeline area), else through D.rows_part
  int ks;          // split-K: work item w = (tile w / ks, K share w % ks); ks > 1 only when the tiles do not
                   // fill the GPU (CG = 1): the shares' fp32 partials meet in D.rows_part (counters
                   // D.rows_cnt), each share sums one slice of the tile's units in share order and runs the
                   // cell epilogue on it (r_split_reduce)
};
constexpr int kRowsMaxItems = 296;     // split work items (tiles x shares) with partial slots
constexpr int kRowsMaxKs = 8;
// K share q of ks over nkb k-blocks: [lo, hi)
__host__ __device__ __forceinline__ void r_kshare(int nkb, int q, int ks, int& lo, int& hi) {
  lo = (int)(((long long)nkb * q) / ks);
  hi = (int)(((long long)nkb * (q + 1)) / ks);
}

__device__ __forceinline__ void rwait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  unsigned long long t0 = 0;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    const unsigned long long now = gtime();
    if (t0 == 0) t0 = now;
    else if (now - t0 > 4000000000ull) __trap();
  }
}

__device__ __forceinline__ uint64_t r_desc(uint32_t saddr) {   // K-major SW128, SBO 1 KB
  return ((uint64_t)((1024u >> 4) | (1u << 14) | (2u << 29)) << 32) | (((saddr >> 4) & 0x3FFF) | (1u << 16));
}

// 4 consecutive TMEM columns of this thread's lane, no wait (the caller waits once)
__device__ __forceinline__ void tld4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int E> struct RAcc { static constexpr int NE = 1; };
template <> struct RAcc<EPI_FC_BWD> { static constexpr int NE = 2; };
template <> struct RAcc<EPI_LSTM_XPROJ> { static constexpr int NE = 4; };
// accumulator layout kind of an epilogue: the eager x-projection (r02) is laid out like one child slot of
// the Tree-LSTM forward (i, o, u, f blocks of UG units) or like the Tree-FC forward (one block); dX too
template <int E> __host__ __device__ constexpr int r_fetch_kind() {
  return E == EPI_LSTM_XPROJ ? EPI_LSTM_FWD : (E == EPI_FC_XPROJ || E == EPI_DX) ? EPI_FC_FWD : E;
}

// accumulators of the VW units at unit offset u (within the tile) -> acc[NE]; VW in {4, 8}
template <int VW>
__device__ __forceinline__ void tldv(uint32_t taddr, uint32_t* r) {
  tld4(taddr, r);
  if constexpr (VW == 8) tld4(taddr + 4, r + 4);
}
template <int E, int NM, int VW>
__device__ __forceinline__ void fetch_acc(uint32_t tb, int UG, int u, FV<VW>* acc) {
  if constexpr (E == EPI_FC_FWD) {
    uint32_t r[VW];
    tldv<VW>(tb + u, r);
    tld_wait();
#pragma unroll
    for (int e = 0; e < VW; ++e) acc[0].v[e] = __uint_as_float(r[e]);
  } else if constexpr (E == EPI_FC_BWD) {
    uint32_t r[2][VW];
    tldv<VW>(tb + u, r[0]);
    tldv<VW>(tb + UG + u, r[1]);
    tld_wait();
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[a].v[e] = __uint_as_float(r[a][e]);
  } else if constexpr (E == EPI_LSTM_FWD) {
    uint32_t r[NM][4][VW];
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int g = 0; g < 4; ++g) tldv<VW>(tb + (uint32_t)(k * 4 * UG + g * UG + u), r[k][g]);
    tld_wait();
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < NM; ++k) s += __uint_as_float(r[k][g][e]);
        acc[g].v[e] = s;
      }
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[3 + k].v[e] = __uint_as_float(r[k][3][e]);
  } else {   // EPI_LSTM_BWD: acc 0 = U_iou^T dz_iou, acc 1 + k = U_f^T dz_fk
    uint32_t r[1 + NM][VW];
#pragma unroll
    for (int a = 0; a < 1 + NM; ++a) tldv<VW>(tb + (uint32_t)(a * UG + u), r[a]);
    tld_wait();
#pragma unroll
    for (int a = 0; a < 1 + NM; ++a)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[a].v[e] = __uint_as_float(r[a][e]);
  }
}

__device__ __forceinline__ uint32_t r_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void r_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA 2-D tile load; CG = 2: completes on the pair leader's barrier (same offset, peer bit cleared)
template <int CG>
__device__ __forceinline__ void r_tma(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  if constexpr (CG == 1) {
    ptx::tma_load_2d(dst, m, c0, c1, bar);
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(ptx::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1),
          "r"(ptx::smem_u32(bar) & kPeerMask)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void r_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1) {
    ptx::mma_bf16(d, a, b, idesc, acc);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}
// arrive on `bar` of this CTA (CG = 1) or of both CTAs of the pair (CG = 2) when the issued MMAs finish
template <int CG>
__device__ __forceinline__ void r_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    ptx::mma_commit(bar);
  } else {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
        ::"r"(ptx::smem_u32(bar)) : "memory");
  }
}

__device__ __forceinline__ void tst16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])),
        "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])) : "memory");
}

// Split-K meeting point of work item (tile j, share kq), called by the 8 epilogue warps (thread = TMEM
// lane r x column half hh) once the share's accumulator is complete.  Every share stores its fp32
// partial (slot layout [item][column][128 lanes]: a warp writes 128 contiguous bytes per column), the
// ks shares of the tile wait for each other (all work items are co-resident: ks x tiles <= #SMs, one
// CTA per SM), then share kq sums the slots in share order (deterministic) for its own slice of the
// tile's units -- columns blk UG + [kq UG/ks, (kq+1) UG/ks) of every accumulator block -- into its TMEM,
// and runs the cell epilogue on that slice: the reduction and the epilogue are spread over all shares.
template <class P_t>
__device__ __forceinline__ void r_split_reduce(const Dev& D, const P_t& P, uint32_t tb, int j, int kq, int r, int hh) {
  // partial slot layout [item][column][128 lanes]: a warp stores / loads 128 contiguous bytes per
  // column (measured faster than per-thread float4 rows: 4x fewer memory requests per instruction)
  const int half = P.acc_cols / 2, c0 = hh * half;
  float* part = D.rows_part;
  const size_t slot = (size_t)128 * P.acc_cols;
  for (int c = c0; c < c0 + half; c += 16) {
    float v[16];
    ptx::tmem_ld16(tb + (uint32_t)c, v);
    float* dst = part + (size_t)(j * P.ks + kq) * slot + (size_t)c * 128 + r;
#pragma unroll
    for (int i = 0; i < 16; ++i) __stcg(dst + (size_t)i * 128, v[i]);
  }
  __threadfence();
  ptx::named_bar_sync(1, 256);
  if (threadIdx.x == 64) {                             // arrive, then wait for the tile's other shares
    int* arrive = D.rows_cnt + 2 * j;
    atomicAdd(arrive, 1);
    unsigned long long t0 = 0;
    while (ptx::ld_acquire_gpu(reinterpret_cast<const uint32_t*>(arrive)) < (uint32_t)P.ks) {
      const unsigned long long now = gtime();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  ptx::named_bar_sync(1, 256);
  __threadfence();
  const int sw = P.UG / P.ks, s0 = kq * sw;            // this share's units [s0, s0 + sw)
  const int nblk = P.acc_cols / P.UG, nch = nblk * (sw / 16);
  const float* base = part + (size_t)(j * P.ks) * slot + r;
  for (int ch = hh; ch < nch; ch += 2) {
    const int c = (ch / (sw / 16)) * P.UG + s0 + (ch % (sw / 16)) * 16;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
    for (int q0 = 0; q0 < P.ks; q0 += 2) {             // two shares' loads in flight, summed in share order
      float x[2][16];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
        if (q0 + qq < P.ks) {
          const float* src = base + (size_t)(q0 + qq) * slot + (size_t)c * 128;
#pragma unroll
          for (int i = 0; i < 16; ++i) x[qq][i] = __ldcg(src + (size_t)i * 128);
        }
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
        if (q0 + qq < P.ks) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += x[qq][i];
        }
    }
    tst16(tb + (uint32_t)c, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  ptx::tc_fence_before();
  ptx::named_bar_sync(1, 256);                         // both halves' columns stored; partials all read
  ptx::tc_fence_after();
  if (threadIdx.x == 64) {                             // the last share out resets the tile's counters
    int* arrive = D.rows_cnt + 2 * j;
    if (atomicAdd(arrive + 1, 1) == P.ks - 1) { arrive[0] = 0; arrive[1] = 0; }
  }
}

// Split-K meeting point through distributed shared memory: the ks shares of tile j are one cluster
// (rank = share).  Each share stages its fp32 partial in its own (drained) pipeline smem as
// [column][128 lanes], the shares meet at a cluster-scope mbarrier (one release-arrive per peer), then
// share kq sums its unit slice over the shares' smem in share order (ld.shared::cluster) into its TMEM.
// The CTAs leave through a full cluster barrier at the end of the kernel (no peer reads a departed CTA).
template <class P_t>
__device__ __forceinline__ void r_split_dsmem(const P_t& P, uint8_t* smem, uint64_t* xbar, uint32_t tb, int kq, int r,
                                              int hh) {
  const int half = P.acc_cols / 2, c0 = hh * half;
  float* sp = reinterpret_cast<float*>(smem);
  for (int c = c0; c < c0 + half; c += 16) {
    float v[16];
    ptx::tmem_ld16(tb + (uint32_t)c, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) sp[(size_t)(c + i) * 128 + r] = v[i];
  }
  ptx::named_bar_sync(1, 256);
  if (threadIdx.x == 64) {
    for (int q = 0; q < P.ks; ++q) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(ptx::smem_u32(xbar)), "r"(q));
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
    }
    const uint32_t a = ptx::smem_u32(xbar);
    unsigned long long t0 = 0;
    for (;;) {
      uint32_t ok;
      asm volatile(
          "{\n\t.reg .pred P;\n\t"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
          "selp.b32 %0, 1, 0, P;\n\t}"
          : "=r"(ok) : "r"(a), "r"(0) : "memory");
      if (ok) break;
      const unsigned long long now = gtime();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) __trap();
    }
  }
  ptx::named_bar_sync(1, 256);
  const int sw = P.UG / P.ks, s0 = kq * sw;            // this share's units [s0, s0 + sw)
  const int nblk = P.acc_cols / P.UG, nch = nblk * (sw / 16);
  const uint32_t base = ptx::smem_u32(sp) + (uint32_t)r * 4u;
  for (int ch = hh; ch < nch; ch += 2) {
    const int c = (ch / (sw / 16)) * P.UG + s0 + (ch % (sw / 16)) * 16;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
    for (int qq = 0; qq < P.ks; ++qq) {                 // share order: deterministic
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + (uint32_t)c * 512u), "r"(qq));
      float x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x[i]) : "r"(ra + (uint32_t)i * 512u) : "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += x[i];
    }
    tst16(tb + (uint32_t)c, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  ptx::tc_fence_before();
  ptx::named_bar_sync(1, 256);
  ptx::tc_fence_after();
}

// x-projection / dX: does row tile [p0, p0 + 128) hold a row that needs the epilogue (a level-0 vertex
// for the x-projection, a pull record for both; k_pull's per-64-row flags)
template <int E>
__device__ __forceinline__ bool r_tile_active(const Dev& D, int p0) {
  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ || E == EPI_DX) {
    if (E != EPI_DX && p0 < dev_lp1(D)) return true;
    return D.tile_x[p0 >> 6] || D.tile_x[(p0 >> 6) + 1];
  } else {
    return true;
  }
}

// SPLIT: the split-K instantiation (P.ks > 1); the plain one keeps ks = 1 at compile time
template <int E, int NM, int QB, int CG, bool SPLIT>
__global__ void __launch_bounds__(kRThreads, 1)
k_rows(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB0,
       const __grid_constant__ CUtensorMap mB1, Dev D, const __grid_constant__ RPlan P) {
  constexpr int NE = E == EPI_LSTM_FWD ? 3 + NM : E == EPI_LSTM_BWD ? 1 + NM : RAcc<E>::NE;
  constexpr int FE = r_fetch_kind<E>();                 // accumulator layout
  constexpr int FNM = E == EPI_LSTM_XPROJ ? 1 : NM;      // (x-projection: one "child slot" of 4 gates)
  // x-projection / dX (r02): row tiles without any row needing the epilogue are skipped by every role
  constexpr bool XD = E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ || E == EPI_DX;
  extern __shared__ __align__(16) uint8_t r_raw[];
  uint8_t* smem = r_raw + ((1024u - (ptx::smem_u32(r_raw) & 1023u)) & 1023u);
  const int S = P.S;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * P.stage);
  uint64_t* empty = full + kRSMax;
  uint64_t* accf = empty + kRSMax;
  uint64_t* acce = accf + 2;
  uint64_t* xbar = acce + 2;                            // split-K DSMEM exchange (cluster scope)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KS = SPLIT ? P.ks : 1;                      // split-K shares per tile
  // debug trace (CAVS_TRACE=1): [0] start, [1] producer past the PDL wait, [2] first stage landed,
  // [3] first accumulator complete, [4] split-K reduction done, [5] first epilogue done
  __shared__ unsigned long long s_tr[6];
  if (D.trace && threadIdx.x == 0) { s_tr[0] = gtime(); s_tr[1] = s_tr[2] = s_tr[3] = s_tr[4] = s_tr[5] = 0; }
  const int rank = CG == 2 ? (int)r_cluster_rank() : 0;
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG, nunits = gridDim.x / CG;   // CTA pair (CG = 2) or CTA

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&accf[b], 1); ptx::mbar_init(&acce[b], 8 * CG); }
    if (SPLIT) ptx::mbar_init(xbar, P.ks);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      ptx::tmem_alloc<512>(tmem_slot);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ptx::smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) r_cluster_sync();             // barriers + TMEM of both CTAs ready
  else if (SPLIT && P.dsm) r_cluster_sync();           // the shares' exchange barriers ready
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer ----
    // one box per lane (lane 0: A, lanes 1..: this CTA's B boxes): boxes issued by one thread are
    // serviced one after another, boxes of different threads in parallel
    if (lane == 0) { ptx::tma_prefetch(&mA); ptx::tma_prefetch(&mB0); ptx::tma_prefetch(&mB1); }
    ptx::griddep_wait();                                 // task rows come from the previous kernels
    if (lane == 0) ptx::griddep_launch();                // PDL: the next task's CTAs may start their prologue
    if (D.trace && lane == 0) s_tr[1] = gtime();
    if (lane <= 4) {
      int step = 0;
      for (int w = unit; w < P.ntiles * KS; w += nunits) {
        const int j = w / KS, kq = w % KS;
        const int p0 = P.lo + (j / P.nut) * 128 * CG + 128 * rank, u0 = (j % P.nut) * P.UG;
        if (XD && !r_tile_active<E>(D, p0)) continue;
        for (int sg = 0; sg < P.nseg; ++sg) {
          const RSeg& Sg = P.seg[sg];
          const CUtensorMap* mb = Sg.bmap ? &mB1 : &mB0;
          const int own = Sg.nbox / CG;                  // this CTA's B boxes: [rank own, +own)
          int kb0, kb1;
          r_kshare(Sg.nkb, kq, KS, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb, ++step) {
            const int s = step % S;
            if (lane > own) continue;
            if (step >= S) rwait(&empty[s], ((step / S) & 1) ^ 1);
            uint8_t* st = smem + s * P.stage;
#ifdef CAVS_ROWS_NOTMA
            if (lane == 0 && leader) ptx::mbar_arrive(&full[s]);       // A/B only: MMA on stale smem
            (void)st; (void)mb; (void)p0; (void)u0;
#else
            if (lane == 0) {
              if (leader) ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)(CG * P.stage));
              r_tma<CG>(st, &mA, Sg.a_col + kb * 64, p0, &full[s]);
            } else {
              const int g = rank * own + lane - 1;
              r_tma<CG>(st + kRA + (lane - 1) * Sg.box_rows * 128, mb, kb * 64, Sg.b_row0[g] + u0, &full[s]);
            }
#endif
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA issuer (the pair's rank-0 CTA) ----
    if (lane == 0 && leader) {
      const uint32_t idesc = ptx::idesc_bf16(128 * CG, P.n, 0, 0);
      int step = 0;
      if (XD) ptx::griddep_wait();                       // k_pull's tile flags
      for (int w = unit, k = 0; w < P.ntiles * KS; w += nunits) {
        const int kq = w % KS;
        if (XD && !r_tile_active<E>(D, P.lo + (w / KS / P.nut) * 128 * CG + 128 * rank)) continue;
        const int buf = P.nbuf == 2 ? (k & 1) : 0;
        const int use = P.nbuf == 2 ? (k >> 1) : k;       // earlier uses of this buffer
        if (use > 0) rwait(&acce[buf], (use - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t tb = tmem + (uint32_t)(buf * P.acc_cols);
        for (int sg = 0; sg < P.nseg; ++sg) {
          const RSeg& Sg = P.seg[sg];
          int kb0, kb1;
          r_kshare(Sg.nkb, kq, KS, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb, ++step) {
            const int s = step % S;
            rwait(&full[s], (step / S) & 1);
            ptx::tc_fence_after();
            if (D.trace && step == 0) s_tr[2] = gtime();
            const uint32_t a = ptx::smem_u32(smem + s * P.stage), b = a + kRA;
#ifndef CAVS_ROWS_NOMMA
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              r_mma<CG>(tb + (uint32_t)Sg.acc_col, r_desc(a + kk * 32), r_desc(b + kk * 32), idesc,
                        (kb != kb0 || kk) ? 1u : 0u);
#else
            (void)a; (void)b; (void)idesc;                   // A/B only: TMA stream without MMAs
#endif
            r_commit<CG>(&empty[s]);
          }
        }
        r_commit<CG>(&accf[buf]);
        ++k;
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: thread = task row (TMEM lane 32q + lane) x half of the tile's units ----
    const int q = warp & 3, hh = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int qpt = P.UG / 8;                            // quads per thread
    uint32_t acce_remote[2] = {0, 0};
    if constexpr (CG == 2) {
      for (int b = 0; b < 2; ++b)
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(acce_remote[b]) : "r"(ptx::smem_u32(&acce[b])));
    }
    ptx::griddep_wait();
    for (int w = unit, k = -1; w < P.ntiles * KS; w += nunits) {
      const int j = w / KS;
      const int p0 = P.lo + (j / P.nut) * 128 * CG + 128 * rank, u0 = (j % P.nut) * P.UG;
      if (XD && !r_tile_active<E>(D, p0)) continue;
      ++k;
      const int p = p0 + r;
      bool valid = p < P.hi;
      VMeta m;
      if (valid) load_meta(D, p, epi_needs_children<E>(), m);
      if (XD && valid) valid = row_active<E>(D, p, m.xrow);
      const int buf = P.nbuf == 2 ? (k & 1) : 0;
      const int use = P.nbuf == 2 ? (k >> 1) : k;
      rwait(&accf[buf], use & 1);
      ptx::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * P.acc_cols);
      // split-K: the shares of the tile meet, share kq finishes the units [kq UG/ks, (kq+1) UG/ks)
      if (D.trace && threadIdx.x == 64 && k == 0) s_tr[3] = gtime();
      if constexpr (SPLIT) {
        if (P.dsm) r_split_dsmem(P, smem, xbar, tb, w % KS, r, hh);
        else r_split_reduce(D, P, tb, j, w % KS, r, hh);
      }
      if (D.trace && threadIdx.x == 64 && k == 0) s_tr[4] = gtime();
      const int sw = P.UG / KS;                        // units finished by this work item
      const int ub = (w % KS) * sw + hh * (sw / 2);    // this thread's first unit within the tile
      // VW units per item: 8 (one 32-byte sector per row and output stream: 256-bit accesses)
      constexpr int VW = 8;
      const int ipt = sw / 2 / VW;                       // items per thread
      if constexpr (E == EPI_LSTM_BWD) {
        // Tree-LSTM backward: the children's dF one child at a time (its state in registers, 8 units
        // per access), the gradient sent to child k = dh~ + U_f^T dz_fk (cells.cuh EpiK)
        const int h = D.h, G = 3 + D.N;
#pragma unroll 1
        for (int it = 0; it < ipt; ++it) {
          const int uo = ub + it * VW, jj = u0 + uo;
          FV<VW> acc[NE];
          fetch_acc<FE, FNM, VW>(tb, P.UG, uo, acc);
#ifndef CAVS_ROWS_NOEPI
          if (valid) {
            const FV<VW> dcbp = ldv<VW>(D.dcb + (size_t)m.p * h + jj);
#pragma unroll
            for (int k = 0; k < NM; ++k) {
              if (k >= m.deg) break;
              const FV<VW> fpk = ldv<VW>(D.gates + (size_t)m.p * G * h + (3 + k) * h + jj);
              LstmChildIn<VW, NM> cin;
              lstm_child_load<VW, NM>(D, jj, m.ch[k], m.ch_vid[k], m.ch_deg[k], cin);
              FV<VW> dh, dc;
#pragma unroll
              for (int e = 0; e < VW; ++e) {
                dh.v[e] = acc[0].v[e] + acc[1 + k].v[e] + cin.dho.v[e];
                dc.v[e] = dcbp.v[e] * fpk.v[e];
              }
              lstm_child_store<__nv_bfloat16, VW, NM>(D, jj, m.ch[k], m.ch_deg[k], dh, dc, cin);
            }
          }
#else
          if (valid && acc[0].v[0] == 12345.f) D.h_out[0] = acc[NE - 1].v[3];
#endif
        }
      } else
#pragma unroll 1
      for (int qb = 0; qb < ipt; qb += QB) {
        typename EpiK<E>::template In<VW, NM> in[QB];
        UnitC<VW> uc[QB];
        if (valid) {
#pragma unroll
          for (int b = 0; b < QB; ++b) {
            const int jj = u0 + ub + (qb + b) * VW;
            EpiK<E>::template load<VW, NM>(D, jj, m, in[b]);
            uc[b] = epi_uses_bias<E>() ? load_unit<VW>(D, jj, epi_is_lstm<E>()) : UnitC<VW>{};
          }
        }
        FV<VW> acc[QB][NE];
#pragma unroll
        for (int b = 0; b < QB; ++b) fetch_acc<FE, FNM, VW>(tb, P.UG, ub + (qb + b) * VW, acc[b]);
#ifndef CAVS_ROWS_NOEPI
        if (valid) {
#pragma unroll
          for (int b = 0; b < QB; ++b)
            EpiK<E>::template store<__nv_bfloat16, VW, NM>(D, u0 + ub + (qb + b) * VW, m, acc[b], in[b], uc[b]);
        }
#else
        if (valid && acc[0][0].v[0] == 12345.f) D.h_out[0] = acc[QB - 1][NE - 1].v[3];   // A/B only: no epilogue stores
#endif
      }
      if (D.trace && threadIdx.x == 64 && k == 0) s_tr[5] = gtime();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {                                   // this warp drained its TMEM lanes
        if (CG == 1 || leader) ptx::mbar_arrive(&acce[buf]);
        else asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acce_remote[buf]) : "memory");
      }
    }
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) r_cluster_sync();             // the peer's last MMA / arrivals are done
  else if (SPLIT && P.dsm) r_cluster_sync();           // no share leaves while a peer reads its smem
  else __syncthreads();
  if (D.trace && threadIdx.x == 0) {
    const unsigned long long at = 8 + 8 * atomicAdd(D.trace, 1ull);
    if (at + 8 < (4u << 20) / 8) {
      D.trace[at] = 7000 + E; D.trace[at + 1] = blockIdx.x | ((unsigned long long)P.lo << 20);
      for (int i = 0; i < 5; ++i) D.trace[at + 2 + i] = s_tr[i + 1] ? s_tr[i + 1] - s_tr[0] : 0;
      D.trace[at + 7] = s_tr[0] | 0;  // start (absolute)
    }
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (CG == 1) ptx::tmem_dealloc<512>(tmem);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// =====================================================================================
// host side
// =====================================================================================
struct RowsState {
  CUtensorMap A_hk, A_dz;
  CUtensorMap B_fwd, B_bwd0, B_bwd1;
  RPlan fwd{}, bwd{};
  // r02: the eager x-projection and pull's adjoint dX on the same kernel (persistent over row tiles,
  // double-buffered accumulators, 256-bit epilogue), rows without an epilogue skipped per 128-row tile
  CUtensorMap A_xp, B_x, B_dx;
  RPlan xp{}, dx{};
  bool xd = false;
  int num_sms = 148;
  int cg = 1;                          // CTAs per MMA: 2 = CTA pairs (cta_group::2, opt-in), 1 = single CTA
  bool can_split = false;              // split-K partial slots carved (D.rows_part) and not disabled
  bool lstm = false;
  bool dsm = false;                    // split-K partials through DSMEM (CAVS_ROWS_DSM=1; measured no faster
                                       // than the global slots at cfg5, profiles/r02_fp32tc.md)
  bool sel_items = false;              // rows_tiles counts work items (tiles x shares) instead of tiles
};

// split-K shares of a task of ntiles tiles: only when the tiles leave SMs idle (CG = 1); every segment
// keeps >= 2 k-blocks per share; at most kRowsMaxItems work items (partial slots)
static int r_ks(const RowsState* rs, const RPlan& P, int ntiles) {
  if (rs->cg != 1 || !rs->can_split || ntiles >= rs->num_sms || ntiles < 1) return 1;
  int min_nkb = 1 << 30;
  for (int sg = 0; sg < P.nseg; ++sg) min_nkb = std::min(min_nkb, P.seg[sg].nkb);
  int ks = std::max(1, std::min({kRowsMaxKs, rs->num_sms / ntiles, min_nkb / 2, kRowsMaxItems / ntiles}));
  // every share finishes a slice of UG / ks units: a whole number of 16-column chunks per column half
  // and of epilogue rounds (QB items of 8 units: 2 for Tree-FC, 1 for Tree-LSTM)
  const int qb = rs->lstm ? 1 : 2;
  while (ks > 1 && (P.UG % ks || (P.UG / ks) % (16 * qb))) --ks;
  return ks;
}

static PFN_cuTensorMapEncodeTiled_v12000 r_enc = nullptr;

static bool renc(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return r_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static RSeg rseg(int a_col, int bmap, int nbox, int box_rows, const int* rows0, int nkb, int acc_col) {
  RSeg S{};
  S.a_col = a_col; S.bmap = bmap; S.nbox = nbox; S.box_rows = box_rows;
  for (int g = 0; g < nbox; ++g) S.b_row0[g] = rows0[g];
  S.nkb = nkb; S.acc_col = acc_col;
  return S;
}

static int r_smem(const RPlan& P) { return 1024 + P.S * P.stage + (2 * kRSMax + 5) * 8 + 16; }

template <int E, int NM, int QB, int CG>
static bool r_attr(const RPlan& P) {
  const bool ok = cudaFuncSetAttribute(k_rows<E, NM, QB, CG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       r_smem(P)) == cudaSuccess;
  if constexpr (CG == 1)
    return ok && cudaFuncSetAttribute(k_rows<E, NM, QB, CG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      r_smem(P)) == cudaSuccess;
  return ok;
}

// Plan of one pass: segments, stage size and depth for CG CTAs per MMA.  CG = 2 splits every
// segment's B rows between the pair (a single 128-row box becomes two 64-row half boxes).
static void r_finish(RPlan& P, int h, int CG) {   // h: the units the tiles cover (the output width)
  if (CG == 2)
    for (int sg = 0; sg < P.nseg; ++sg) {
      RSeg& S = P.seg[sg];
      if (S.nbox == 1) {
        S.nbox = 2; S.b_row0[1] = S.b_row0[0] + S.box_rows / 2; S.box_rows /= 2;
      }
    }
  P.stage = kRA + P.n / CG * 128;
  P.S = std::min(kRSMax, (232448 - 2048 - (2 * kRSMax + 5) * 8 - 16) / P.stage);
  P.nbuf = 2 * P.acc_cols <= 512 ? 2 : 1;
  P.nut = h / P.UG;
}

RowsState* rows_init(const Dev& D, int max_vertices) {
  const char* env = std::getenv("CAVS_ROWS");
  if (env && env[0] == '0') return nullptr;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int h = D.h, N = D.N;
  if (lstm && (h % 128 || N > 2)) return nullptr;
  if (!lstm && h % 256) return nullptr;
  if (!r_enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return nullptr;
    r_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  RowsState* rs = new RowsState();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&rs->num_sms, cudaDevAttrMultiProcessorCount, dev);
  // CTA pairs are opt-in (CAVS_ROWS_PAIR=1): measured at cfg5 they do not beat one CTA per MMA
  // (the pair's TMA stream runs in lockstep on the slower SM; profiles/r02_rows.md)
  const char* pe = std::getenv("CAVS_ROWS_PAIR");
  rs->cg = (pe && pe[0] == '1') ? 2 : 1;
  const char* ke = std::getenv("CAVS_ROWS_KSPLIT");
  rs->can_split = D.rows_part && D.rows_cnt && !(ke && ke[0] == '0');
  rs->lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const char* de = std::getenv("CAVS_ROWS_DSM");
  rs->dsm = de && de[0] == '1';
  const char* se = std::getenv("CAVS_ROWS_SEL");
  rs->sel_items = se ? se[0] == 'i' : !rs->lstm;
  const int CG = rs->cg;
  const uint64_t Vp = (uint64_t)max_vertices + kPadRows, G = lstm ? 3 + N : 1;
  bool ok = renc(&rs->A_hk, D.Hk, (uint64_t)N * h, Vp, 128) && renc(&rs->A_dz, D.dZ, G * h, Vp, 128);
  RPlan& F = rs->fwd;
  RPlan& B = rs->bwd;
  if (lstm) {
    // forward: block k (4 x 64 columns) = (U_i, U_o, U_u, U_f) h_k for 64 units
    F.UG = 64; F.n = 256; F.nseg = N;
    const int rows4[4] = {0, h, 2 * h, 3 * h};
    for (int k = 0; k < N; ++k) F.seg[k] = rseg(k * h, 0, 4, 64, rows4, h / 64, k * 256);
    F.acc_cols = 256 * N;
    ok = ok && renc(&rs->B_fwd, D.Wa, h, 4 * (uint64_t)h, 64);                  // U4 [4h x h]
    // backward: acc 0 = U_iou^T dz_iou (K = 3h), acc 1 + k = U_f^T dz_fk (K = h); 128 units
    B.UG = 128; B.n = 128; B.nseg = 1 + N;
    const int r0[1] = {0};
    B.seg[0] = rseg(0, 0, 1, 128, r0, 3 * h / 64, 0);
    for (int k = 0; k < N; ++k) B.seg[1 + k] = rseg((3 + k) * h, 1, 1, 128, r0, h / 64, (1 + k) * 128);
    B.acc_cols = 128 * (1 + N);
    const uint32_t br = CG == 2 ? 64 : 128;                                       // pair: half boxes
    ok = ok && renc(&rs->B_bwd0, D.Wc, 3 * (uint64_t)h, h, br) && renc(&rs->B_bwd1, D.Wd, h, h, br);
  } else {
    // forward: z = [h_l | h_r] W_c^T for 256 units
    F.UG = 256; F.n = 256; F.nseg = 1;
    const int r01[2] = {0, 128};
    F.seg[0] = rseg(0, 0, 2, 128, r01, 2 * h / 64, 0);
    F.acc_cols = 256;
    ok = ok && renc(&rs->B_fwd, D.Wa, 2 * (uint64_t)h, h, 128);                 // W_c [h x 2h]
    // backward: (dh_l, dh_r) = dz W_c for 128 units: W_c^T rows u0 and h + u0
    B.UG = 128; B.n = 256; B.nseg = 1;
    const int r2[2] = {0, h};
    B.seg[0] = rseg(0, 0, 2, 128, r2, h / 64, 0);
    B.acc_cols = 256;
    ok = ok && renc(&rs->B_bwd0, D.Wc, h, 2 * (uint64_t)h, 128);                // W_c^T [2h x h]
    rs->B_bwd1 = rs->B_bwd0;
  }
  r_finish(F, h, CG);
  r_finish(B, h, CG);
  // x-projection (Z = X W^T over the pulled rows) and dX = dZ W: single-CTA tiles (CG = 1 only)
  const int d = D.d;
  // default on for Tree-FC (cfg5: x-projection 210 -> 167 us, dX 176 -> 125 us); the Tree-LSTM
  // x-projection measured slower than gemm.cu's (its epilogue writes five arenas per unit, and the
  // 2-CTA-per-SM row GEMM overlaps two epilogues), so CAVS_ROWS_XD=1 opts it in, =0 turns both off
  const char* xe = std::getenv("CAVS_ROWS_XD");
  const bool xd_on = xe ? xe[0] == '1' : !lstm;
  rs->xd = CG == 1 && xd_on && d % 256 == 0;
  if (rs->xd) {
    RPlan& X = rs->xp;
    RPlan& Q = rs->dx;
    bool okx = renc(&rs->A_xp, D.Xp, (uint64_t)d, Vp, 128);
    if (lstm) {
      X.UG = 64; X.n = 256; X.nseg = 1;
      const int rows4[4] = {0, h, 2 * h, 3 * h};
      X.seg[0] = rseg(0, 0, 4, 64, rows4, d / 64, 0);
      okx = okx && renc(&rs->B_x, D.Wb, (uint64_t)d, 4 * (uint64_t)h, 64);          // W4 [4h x d]
      okx = okx && renc(&rs->B_dx, D.We, G * h, (uint64_t)d, 128);                   // WT [d x G h]
    } else {
      X.UG = 256; X.n = 256; X.nseg = 1;
      const int r01[2] = {0, 128};
      X.seg[0] = rseg(0, 0, 2, 128, r01, d / 64, 0);
      okx = okx && renc(&rs->B_x, D.Wb, (uint64_t)d, h, 128);                        // Wx [h x d]
      okx = okx && renc(&rs->B_dx, D.We, (uint64_t)h, (uint64_t)d, 128);             // WxT [d x h]
    }
    X.acc_cols = 256;
    Q.UG = 256; Q.n = 256; Q.nseg = 1;
    const int r01[2] = {0, 128};
    Q.seg[0] = rseg(0, 0, 2, 128, r01, (int)(G * h) / 64, 0);
    Q.acc_cols = 256;
    r_finish(X, h, 1);
    r_finish(Q, d, 1);
    rs->xd = okx;
  }
  auto attrs = [&](auto cg) {
    constexpr int C = decltype(cg)::value;
    if (lstm)
      return N == 1 ? r_attr<EPI_LSTM_FWD, 1, 1, C>(F) && r_attr<EPI_LSTM_BWD, 1, 1, C>(B)
                    : r_attr<EPI_LSTM_FWD, 2, 1, C>(F) && r_attr<EPI_LSTM_BWD, 2, 1, C>(B);
    return r_attr<EPI_FC_FWD, 1, 2, C>(F) && r_attr<EPI_FC_BWD, 1, 2, C>(B);
  };
  ok = ok && (CG == 2 ? attrs(std::integral_constant<int, 2>{}) : attrs(std::integral_constant<int, 1>{}));
  if (ok && rs->xd) {
    bool okx;
    if (lstm)
      okx = (N == 1 ? r_attr<EPI_LSTM_XPROJ, 1, 1, 1>(rs->xp) : r_attr<EPI_LSTM_XPROJ, 2, 1, 1>(rs->xp)) &&
            r_attr<EPI_DX, 1, 2, 1>(rs->dx);
    else
      okx = r_attr<EPI_FC_XPROJ, 1, 2, 1>(rs->xp) && r_attr<EPI_DX, 1, 2, 1>(rs->dx);
    rs->xd = okx;
  }
  if (!ok) { delete rs; return nullptr; }
  return rs;
}

void rows_destroy(RowsState* rs) { delete rs; }

// a task's size measure for the caller's "use the row-tiled kernel" threshold: its tiles, or (Tree-FC,
// or CAVS_ROWS_SEL=items) its work items = tiles x split-K shares
int rows_tiles(const RowsState* rs, bool backward, int rows) {
  if (!rs) return 0;
  const RPlan& P = backward ? rs->bwd : rs->fwd;
  const int nt = cdiv(rows, 128 * rs->cg) * P.nut;
  return rs->sel_items ? nt * r_ks(rs, P, nt) : nt;
}

int rows_pair(const RowsState* rs) { return rs ? rs->cg : 0; }

template <int E, int NM, int QB, int CG>
static void r_launch(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1, const Dev& D, const RPlan& P,
                     int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kRThreads, 1, 1);
  cfg.dynamicSmemBytes = r_smem(P);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;          // CTA pair on one TPC (CG = 2); split-K shares (DSMEM)
  at[1].val.clusterDim.x = (CG == 1 && P.ks > 1 && P.dsm) ? P.ks : CG;
  at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if constexpr (CG == 1) {
    if (P.ks > 1) { cudaLaunchKernelEx(&cfg, k_rows<E, NM, QB, CG, true>, a, b0, b1, D, P); return; }
  }
  cudaLaunchKernelEx(&cfg, k_rows<E, NM, QB, CG, false>, a, b0, b1, D, P);
}

template <int CG>
static void rows_go(const Dev& D, RowsState* rs, bool backward, RPlan& P, cudaStream_t s) {
  P.ntiles = cdiv(P.hi - P.lo, 128 * CG) * P.nut;
  // split-K when the tiles leave SMs idle: ks shares per tile (every segment keeps >= 2 k-blocks
  // per share), at most kRowsMaxItems work items (partial slots)
  P.ks = r_ks(rs, P, P.ntiles);
  // the DSMEM exchange needs the partial ([acc_cols][128] fp32) to fit the drained pipeline area
  P.dsm = P.ks > 1 && rs->dsm && (size_t)P.acc_cols * 128 * 4 <= (size_t)P.S * P.stage;
  const int grid = std::min(P.ntiles * P.ks * CG, rs->num_sms / CG * CG);
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  if (lstm) {
    if (!backward) {
      if (D.N == 1) r_launch<EPI_LSTM_FWD, 1, 1, CG>(rs->A_hk, rs->B_fwd, rs->B_fwd, D, P, grid, s);
      else r_launch<EPI_LSTM_FWD, 2, 1, CG>(rs->A_hk, rs->B_fwd, rs->B_fwd, D, P, grid, s);
    } else {
      if (D.N == 1) r_launch<EPI_LSTM_BWD, 1, 1, CG>(rs->A_dz, rs->B_bwd0, rs->B_bwd1, D, P, grid, s);
      else r_launch<EPI_LSTM_BWD, 2, 1, CG>(rs->A_dz, rs->B_bwd0, rs->B_bwd1, D, P, grid, s);
    }
  } else {
    if (!backward) r_launch<EPI_FC_FWD, 1, 2, CG>(rs->A_hk, rs->B_fwd, rs->B_fwd, D, P, grid, s);
    else r_launch<EPI_FC_BWD, 1, 2, CG>(rs->A_dz, rs->B_bwd0, rs->B_bwd1, D, P, grid, s);
  }
}

bool rows_xd(const RowsState* rs) { return rs && rs->xd; }

bool rows_xproj(const Dev& D, RowsState* rs, cudaStream_t s) {
  if (!rs || !rs->xd || D.V < 1) return false;
  RPlan P = rs->xp;
  P.lo = 0; P.hi = D.V; P.ks = 1; P.dsm = 0;
  P.ntiles = cdiv(P.hi, 128) * P.nut;
  const int grid = std::min(P.ntiles, rs->num_sms);
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    if (D.N == 1) r_launch<EPI_LSTM_XPROJ, 1, 1, 1>(rs->A_xp, rs->B_x, rs->B_x, D, P, grid, s);
    else r_launch<EPI_LSTM_XPROJ, 2, 1, 1>(rs->A_xp, rs->B_x, rs->B_x, D, P, grid, s);
  } else {
    r_launch<EPI_FC_XPROJ, 1, 2, 1>(rs->A_xp, rs->B_x, rs->B_x, D, P, grid, s);
  }
  return true;
}

bool rows_dx(const Dev& D, RowsState* rs, cudaStream_t s) {
  if (!rs || !rs->xd || !D.dx || D.V < 1) return false;
  RPlan P = rs->dx;
  P.lo = 0; P.hi = D.V; P.ks = 1; P.dsm = 0;
  P.ntiles = cdiv(P.hi, 128) * P.nut;
  const int grid = std::min(P.ntiles, rs->num_sms);
  r_launch<EPI_DX, 1, 2, 1>(rs->A_dz, rs->B_dx, rs->B_dx, D, P, grid, s);
  return true;
}

bool rows_level(const Dev& D, RowsState* rs, bool backward, int lo, int hi, cudaStream_t s) {
  if (!rs || hi <= lo) return false;
  RPlan P = backward ? rs->bwd : rs->fwd;
  P.lo = lo; P.hi = hi;
  if (rs->cg == 2) rows_go<2>(D, rs, backward, P, s);
  else rows_go<1>(D, rs, backward, P, s);
  return true;
}

}  // namespace cavs
