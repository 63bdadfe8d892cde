// persist.cu — BF16 mode: ONE persistent, weight-stationary launch for all batching tasks of a
// pass (Alg. 1 FORWARD / BACKWARD loop; the batched "Batched Execution"
// of §3.5).
//
// Why: a level-by-level launch pays, per task V_t, a kernel launch + a fresh stream of F's
// weights (2-8 MB) through the SMs, and the small tasks at the top of the trees are pure
// latency.  Here every CTA keeps a fixed 128-row slice of the weights resident in TMEM (staged
// once through shared memory by TMA and copied with tcgen05.cp; the MMA takes A from TMEM) for the
// whole pass, and the tasks are separated by a cluster-local barrier instead of kernel boundaries.
//
// Decomposition (swap-AB, like tc.cu): D[row, task] = sum_k A[row, k] B[task, k], M = 128 weight
// rows, N = NT task rows (16/32/64 chosen per task), accumulators in TMEM after the weights.  The
// 128 rows of a CTA are ngrp "row groups" of UG units each, every group a different gate
// (Tree-LSTM: i, o, u, f of the same 32 units, UG = 32; Tree-FC: the two children's blocks of the
// same 64 units, UG = 64), so a CTA owns ALL the gates of its units and the fused cell epilogue
// needs no inter-CTA exchange.  A group only pairs with its own operand columns; where operands
// differ per group (backward: dz_i, dz_o, dz_u, dz_f; Tree-FC forward: h_l, h_r) each operand gets
// its own accumulator and the epilogue keeps the matching group (the Tree-LSTM backward's
// discarded rows: see persist_bwd.cu for the K-split alternative and why it is opt-in).
//
//   grid = nub x R CTAs: R clusters (graph ranges; the graphs of a batch are independent,
//   P:L388-391) of nub = h / UG unit-block CTAs, one CTA per SM; cluster r runs its own rows of
//   every task (table crow[t][r], k_build_maps) and only its CTAs synchronise between tasks
//   (cluster-scope mbarrier, persist_common.cuh).
//   warps 0-2: TMA producers (weights once; then B boxes {64 k, NT rows, sk k-blocks} of the
//              task rows, one warp per pipeline stage), warp 3: TMEM allocator + MMA issuer,
//   warps 4-11: per-vertex metadata, TMEM -> smem staging, fused cell epilogue (cells.cuh),
//              and the cluster task barrier.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "persist.h"
#include "persist_common.cuh"

namespace cavs {

constexpr int kPThreads = 384;       // 12 warps (whole 4-warp register granules: up to 168 regs)
constexpr int kPProd = 3;            // producer warps 0-2, MMA warp 3
constexpr int kPMma = 3;
constexpr int kPEpi0 = 4;            // first epilogue warp
constexpr int kPKb = 16384;          // one resident A k-block: 128 rows x 128 B (SW128, K-major)
constexpr int kPStageMin = 16384;    // B stage granularity (one 16-row x 8 k-block box)
constexpr int kPMaxNT = 64;
constexpr int kPMaxS = 12;           // B pipeline stages (TMEM-resident weights free the smem)

struct PPlan {
  int UG, ngrp, nkbA;                // units per CTA, row groups, resident k-blocks (K = 64 nkbA)
  int grp_row0[4], grp_col0[4];      // A rows grp_row0 + u0 .. + UG, columns grp_col0 + 64 kb
  int nseg, seg_bcol[8], seg_acc[8]; // MMA segments: all resident k-blocks x B columns [bcol, bcol + K)
  int seg_init[8];                   // 1: the segment is the first one writing its accumulator
  int nacc;
  int nslot, slot_grp[8], slot_nacc[8], slot_acc[8][4];   // staged slot = sum of accs, one group
  int ne, e_n[8], e_slot[8][3];      // epilogue accumulator e = sum of slots
  int S;                             // B pipeline stages
  int sk[3];                         // k-blocks per B box (= per stage) for NT = 16 / 32 / 64
  int stage;                         // bytes per B stage (one box); boxes span segments (contiguous B columns)
  int tsA;                           // 1: weights resident in TMEM (A operand from TMEM), 0: in smem
  int acc0;                          // first TMEM column of the accumulators
  int max_ni;                        // largest task tile index (NT = 16 << ni) the TMEM budget admits
  int nub, R;
  int mc;                            // 1: B boxes multicast to the whole cluster (every CTA of a graph
                                     //    range reads the same task rows): one TMA per box per cluster
  int xs_off, meta_off, bar_off;
  int is_bwd;                        // host: backward plan (stage-size override)
};

// Compile-time staging layout per epilogue kind (matches the host plan of persist_init):
// xs slot s holds one row group's accumulator(s); epilogue accumulator e sums slots.
template <int E0, int NM> struct PLay {
  static constexpr int E = epi_base(E0);             // inference kinds: the training kind's layout
  static constexpr bool lstm = E == EPI_LSTM_FWD || E == EPI_LSTM_BWD;
  static constexpr int UG = lstm ? 32 : 64;
  static constexpr int NSLOT = lstm ? 3 + NM : 2;
  static constexpr int NE = E == EPI_LSTM_FWD ? 3 + NM : E == EPI_LSTM_BWD ? 1 + NM : E == EPI_FC_FWD ? 1 : 2;
  static __device__ __forceinline__ constexpr int grp(int s) { return lstm ? (s < 3 ? s : 3) : s; }
  static __device__ __forceinline__ constexpr int nacc(int s) { return E == EPI_LSTM_FWD && s < 3 ? NM : 1; }
  static __device__ __forceinline__ constexpr int acc(int s, int a) {
    return E == EPI_LSTM_FWD ? (s < 3 ? a : s - 3) : E == EPI_FC_BWD ? 0 : s;
  }
  static __device__ __forceinline__ constexpr int e_n(int e) {
    return E == EPI_LSTM_BWD && e == 0 ? 3 : E == EPI_FC_FWD ? 2 : 1;
  }
  static __device__ __forceinline__ constexpr int e_slot(int e, int z) {
    return E == EPI_LSTM_BWD ? (e == 0 ? z : e + 2) : E == EPI_FC_FWD ? z : e;
  }
};

// MMA issue of one task's tiles (NT compile-time: constant instruction descriptor, accumulator
// columns and descriptor strides; only 32-bit adds per tcgen05.mma).
// stage-free arrival: this CTA's MMAs of the stage are done -> the stage's empty barrier of this CTA,
// or (multicast plan) of every CTA of the cluster, since any of them may issue the stage's next box
__device__ __forceinline__ void stage_commit(uint64_t* bar, int mc, uint32_t mask) {
  if (mc)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(ptx::smem_u32(bar)), "h"((uint16_t)mask) : "memory");
  else
    ptx::mma_commit(bar);
}

template <int NT, bool TS>
__device__ __forceinline__ void mma_level(const PPlan& P, int ntile, uint32_t a_lo, uint32_t b_lo,
                                          uint64_t* full, uint64_t* empty, uint64_t* done, uint64_t* tmem_empty,
                                          int& step, int& tcount, unsigned long long* tr) {
  // Whole warp runs the loop (warp-uniform operands live in uniform registers); one elected
  // lane issues each box's MMAs + commit.
  constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
  constexpr int ni = NT == 16 ? 0 : NT == 32 ? 1 : 2;
  // plan constants hoisted into registers (no indexed constant-bank loads in the issue loop);
  // accumulator of segment sg = acc0 + sg * NT (every plan maps segment sg to accumulator sg)
  const int sk = P.sk[ni], S = P.S;
  const int nkbA = P.nkbA;
  const int nkb = P.nseg * nkbA;                    // the tile's k-blocks, segment-major
  const int nbox = (nkb + sk - 1) / sk;
  const uint32_t acc0 = (uint32_t)P.acc0, stage16 = (uint32_t)(P.stage >> 4);
  for (int j = 0; j < ntile; ++j, ++tcount) {
    if (tcount > 0) { pwait_warp(tmem_empty, (tcount - 1) & 1); ptx::tc_fence_after(); }
    int sg = 0, kba = 0;                              // (segment, weight k-block) of the next k-block
    for (int b = 0; b < nbox; ++b, ++step) {
      const int s = step % S;
      pwait_warp(&full[s], (step / S) & 1);
      ptx::tc_fence_after();
      if (tr) { if (tr[0] == 0) tr[0] = gtime(); if (tr[1] == 0) tr[2] = gtime(); }   // first / last box of the first tile
      const int cnt = min(nkb, (b + 1) * sk) - b * sk;
      if (ptx::elect_one()) {
        uint32_t bl = b_lo + (uint32_t)s * stage16;
        int kbi = kba;
        uint32_t d = acc0 + (uint32_t)(sg * NT);
        for (int g = 0; g < cnt; ++g) {
          const uint32_t at = (uint32_t)kbi * 32u;     // TMEM column of the weights' k-block
          const uint32_t al = a_lo + (uint32_t)kbi * (kPKb >> 4);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc_flag = (kk == 0 && kbi == 0) ? 0u : 1u;   // first product into the accumulator
            if constexpr (TS) ptx::mma_bf16_ts(d, at + kk * 8, sw128_desc(bl + kk * 2), idesc, acc_flag);
            else ptx::mma_bf16(d, sw128_desc(al + kk * 2), sw128_desc(bl + kk * 2), idesc, acc_flag);
          }
          bl += (NT * 128) >> 4;
          if (++kbi == nkbA) { kbi = 0; d += NT; }
        }
        stage_commit(&empty[s], P.mc, (1u << P.nub) - 1u);
      }
      __syncwarp();
      kba += cnt;                                     // advance (all lanes, uniform)
      while (kba >= nkbA) { kba -= nkbA; ++sg; }
    }
    if (ptx::elect_one()) ptx::mma_commit(done);
    __syncwarp();
    if (tr && tr[1] == 0) tr[1] = gtime();
  }
}

// nlev < 0 (sync-free mode): the tasks of the pass from the device header (t_first = 1 forward,
// T - 1 backward); an invalid or DAG batch runs no task.  Call after the PDL wait.
__device__ __forceinline__ void resolve_tasks(const Dev& D, int dir, int& t_first, int& nlev) {
  if (nlev >= 0) return;
  const int T = dev_T(D);
  nlev = T > 1 ? T - 1 : 0;
  t_first = dir > 0 ? 1 : T - 1;
}

template <int E, int NE, int NM>
__global__ void __launch_bounds__(kPThreads, 1)
k_persist(const __grid_constant__ CUtensorMap ma0, const __grid_constant__ CUtensorMap ma1,
          const __grid_constant__ CUtensorMap ma2, const __grid_constant__ CUtensorMap ma3,
          const __grid_constant__ CUtensorMap mb16, const __grid_constant__ CUtensorMap mb32,
          const __grid_constant__ CUtensorMap mb64, Dev D, PPlan P, int t_first, int nlev, int dir) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-aligned base by pointer arithmetic on the __shared__ symbol (keeps the shared address
  // space visible to the compiler: LDS/STS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  using L = PLay<E, NM>;
  static_assert(L::NE == NE, "epilogue accumulator count");
  uint8_t* sA = smem;                                           // weights as loaded by TMA
  uint8_t* sB = P.tsA ? smem : smem + P.nkbA * kPKb;            // TMEM weights: stages reuse sA
  float* xs = reinterpret_cast<float*>(smem + P.xs_off);        // [nslot][64][UG]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bar_off);
  uint64_t* empty = full + kPMaxS;
  uint64_t* done = empty + kPMaxS;
  uint64_t* tmem_empty = done + 1;
  uint64_t* abar = tmem_empty + 1;
  uint64_t* acopy = abar + 1;                                   // weights copied smem -> TMEM
  uint64_t* cbar = acopy + 1;                                   // cluster task barrier
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbar + 1);
  int* gate = reinterpret_cast<int*>(tmem_slot + 1);
  __shared__ unsigned long long s_tmax;                          // debug trace only

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ub = blockIdx.x % P.nub, r = blockIdx.x / P.nub;   // cluster rank = unit block, cluster = r
  const int u0 = ub * P.UG;
  const int S = P.S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], P.mc ? P.nub : 1); }
    ptx::mbar_init(done, 1);
    ptx::mbar_init(tmem_empty, 8);
    ptx::mbar_init(abar, P.ngrp);
    ptx::mbar_init(acopy, 1);
    ptx::mbar_init(cbar, P.nub);
    *gate = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kPMma) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  cluster_sync_all();                                 // peers' barriers initialised before any remote arrive
  // PDL: every CTA of this persistent grid is resident from here on, so the next kernel (k_roots after
  // the forward, the lazy GEMMs after the backward) may launch onto the idle SMs and run its prologue;
  // its griddepcontrol.wait still orders every read of this grid's outputs
  if (threadIdx.x == 0) ptx::griddep_launch();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kPProd) {
    // ------------------------------------------------------------------ producers
    if (lane == 0) {
      const int w = warp;
      for (int g = w; g < P.ngrp; g += kPProd) {      // resident weights: group g, all k-blocks
        const CUtensorMap* ma = g == 0 ? &ma0 : g == 1 ? &ma1 : g == 2 ? &ma2 : &ma3;
        ptx::tma_prefetch(ma);
        ptx::mbar_arrive_expect_tx(abar, P.nkbA * P.UG * 128);
        for (int kb = 0; kb < P.nkbA; ++kb)
          ptx::tma_load_2d(sA + kb * kPKb + g * P.UG * 128, ma, P.grp_col0[g] + kb * 64, P.grp_row0[g] + u0, abar);
      }
      ptx::tma_prefetch(&mb16); ptx::tma_prefetch(&mb32); ptx::tma_prefetch(&mb64);
      if (P.tsA) pwait(acopy, 0);                     // stages overlay the weights' staging area
      ptx::griddep_wait();                            // task rows come from the previous kernels
      resolve_tasks(D, dir, t_first, nlev);
      int step = 0;
      for (int i = 0; i < nlev; ++i) {
        const int t = t_first + i * dir;
        int lo, M;
        cl_rows(D, t, r, lo, M);
        const int ni = nt_index(M, 1, P.max_ni), nt = 16 << ni;
        const int ntile = (M + nt - 1) / nt;
        if (ntile == 0) continue;
        const CUtensorMap* mb = ni == 0 ? &mb16 : ni == 1 ? &mb32 : &mb64;
        const int sk = P.sk[ni], nbox = (P.nseg * P.nkbA + sk - 1) / sk;
        const uint32_t bytes = (uint32_t)nt * 128u * (uint32_t)sk;
        if (i > 0) {                                  // previous task finished grid-wide
          const unsigned long long tw = D.trace ? gtime() : 0;
          // acquire: the cluster's task writes are visible.  Back off between polls: the producers wait
          // here through the MMA and epilogue of the previous task, and a tight ld.shared spin competes
          // with the MMAs' shared-memory operand reads (CAVS_GATE_SPIN=1 build: tight spin, A/B)
#ifdef CAVS_GATE_SPIN
          while (gate_get(gate) < i) { }
#else
          while (gate_get(gate) < i) __nanosleep(128);
#endif
          ptx::fence_proxy_async_global();     // ... to this thread's TMA (async proxy) reads
          if (D.trace && w == 0) ptrace(D, 3000 + E, blockIdx.x, i, tw, gtime(), 0, 0, 0);
        }
        if (D.trace && w == 0) ptrace(D, 5000 + E, blockIdx.x, i, gtime(), 0, 0, 0, 0);
        for (int j = 0; j < ntile; ++j) {
          const int p0 = lo + j * nt;
          for (int b = 0; b < nbox; ++b, ++step) {   // one box = sk consecutive k-blocks of the row block
            const int s = step % S;
            if (s % kPProd != w) continue;
            const uint32_t ph = (step / S) & 1;
            if (P.mc) pwait(&empty[s], ph);              // freed by every CTA of the cluster (phase 0: initial)
            else if (step >= S) pwait(&empty[s], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&full[s], bytes);
            if (!P.mc) {
              ptx::tma_load_3d(sB + s * P.stage, mb, 0, p0, P.seg_bcol[0] / 64 + b * sk, &full[s]);
            } else if (step % P.nub == ub) {             // this CTA's turn: one box for the whole cluster
              asm volatile(
                  "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                  " [%0], [%1, {%2, %3, %4}], [%5], %6;"
                  ::"r"(ptx::smem_u32(sB + s * P.stage)), "l"(reinterpret_cast<uint64_t>(mb)), "r"(0), "r"(p0),
                    "r"(P.seg_bcol[0] / 64 + b * sk), "r"(ptx::smem_u32(&full[s])), "h"((uint16_t)((1u << P.nub) - 1u))
                  : "memory");
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kPMma) {
    // ------------------------------------------------------------------ MMA issuer
    {
      // The CTA is alone on its SM (shared memory) and owns all 512 TMEM columns, so the
      // allocation starts at column 0: accumulator addresses are then warp-uniform constants
      // (no per-MMA register->uniform waterfall in the issue loop).
      if (tmem != 0) __trap();
      pwait_warp(abar, 0);
      ptx::tc_fence_after();
      if (P.tsA) {                                    // weights -> TMEM columns [0, 32 nkbA)
        if (ptx::elect_one()) {
          for (int kb = 0; kb < P.nkbA; ++kb)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::tmem_cp_128x256b((uint32_t)(kb * 32 + kk * 8),
                                    sw128_desc(((ptx::smem_u32(sA + kb * kPKb + kk * 32) >> 4) & 0x3FFF) | (1u << 16)));
          ptx::mma_commit(acopy);
        }
        __syncwarp();
        pwait_warp(acopy, 0);
        ptx::tc_fence_after();
      }
      if (P.mc) {
        // multicast plan: a peer may write this CTA's stages only once its weights left the staging
        // area (tcgen05.cp above): the initial phase of every stage's empty barrier, in every CTA,
        // completes with one arrival per CTA, issued when this thread's copies are done
        if (ptx::elect_one())
          for (int s2 = 0; s2 < S; ++s2) stage_commit(&empty[s2], 1, (1u << P.nub) - 1u);
        __syncwarp();
      }
      const uint32_t a_lo = ((ptx::smem_u32(sA) >> 4) & 0x3FFF) | (1u << 16);
      const uint32_t b_lo = ((ptx::smem_u32(sB) >> 4) & 0x3FFF) | (1u << 16);
      ptx::griddep_wait();
      resolve_tasks(D, dir, t_first, nlev);
      int step = 0, tcount = 0;
      for (int i = 0; i < nlev; ++i) {
        const int t = t_first + i * dir;
        int lo, M;
        cl_rows(D, t, r, lo, M);
        const int ni = nt_index(M, 1, P.max_ni), nt = 16 << ni;
        const int ntile = (M + nt - 1) / nt;
        unsigned long long trm[3] = {0, 0, 0};
        unsigned long long* tr = D.trace ? trm : nullptr;
        if (P.tsA) {
          if (ni == 0) mma_level<16, true>(P, ntile, a_lo, b_lo, full, empty, done, tmem_empty, step, tcount, tr);
          else if (ni == 1) mma_level<32, true>(P, ntile, a_lo, b_lo, full, empty, done, tmem_empty, step, tcount, tr);
          else mma_level<64, true>(P, ntile, a_lo, b_lo, full, empty, done, tmem_empty, step, tcount, tr);
        } else {
          if (ni == 0) mma_level<16, false>(P, ntile, a_lo, b_lo, full, empty, done, tmem_empty, step, tcount, tr);
          else if (ni == 1) mma_level<32, false>(P, ntile, a_lo, b_lo, full, empty, done, tmem_empty, step, tcount, tr);
          else mma_level<64, false>(P, ntile, a_lo, b_lo, full, empty, done, tmem_empty, step, tcount, tr);
        }
        if (D.trace && ntile > 0 && lane == 0) ptrace(D, 4000 + E, blockIdx.x, i, trm[0], trm[1], trm[2], nt, 0);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ epilogue (8 warps)
    const int et = threadIdx.x - kPEpi0 * 32;          // 0..255
    const int q = warp & 3, half = (warp - kPEpi0) >> 2;
    constexpr int quads = L::UG / 4;
    const int quad = et % quads;                       // constant: 256 % quads == 0
    const int j = u0 + quad * 4;
    ptx::griddep_wait();
    resolve_tasks(D, dir, t_first, nlev);
    const UnitC<4> uc = epi_uses_bias<E>() ? load_unit<4>(D, j, epi_is_lstm<E>()) : UnitC<4>{};
    constexpr int CH = epi_needs_children<E>() ? 1 : 2;
    int tcount = 0, nbar = 0;
    for (int i = 0; i < nlev; ++i) {
      const int t = t_first + i * dir;
      int lo, M;
      cl_rows(D, t, r, lo, M);
      const int ni = nt_index(M, 1, P.max_ni), nt = 16 << ni;
      const int ntile = (M + nt - 1) / nt;
      unsigned long long tr0 = 0, tr1 = 0, tr2 = 0, tr3 = 0;
      if (D.trace && et == 0) tr0 = gtime();
      if (i > 0 && ntile > 0) {                         // inputs of V_t are final once the barrier passed
#ifdef CAVS_GATE_SPIN
        if (lane == 0) while (gate_get(gate) < i) { }
#else
        if (lane == 0) while (gate_get(gate) < i) __nanosleep(32);
#endif
        __syncwarp();
      }
      for (int jt = 0; jt < ntile; ++jt, ++tcount) {
        const int p0 = lo + jt * nt;
        const int valid = min(nt, lo + M - p0);
        const int items = quads * valid;
        // ---- this thread's first round of (unit quad, column) items: metadata + cell inputs,
        //      loaded while the TMA / MMA of the tile are still in flight ----
        VMeta mt[CH];
        typename EpiK<E>::template In<4, NM> in[CH];
        int base = et;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int it = base + 256 * c;
          if (it < items) {
            load_meta(D, p0 + it / quads, epi_needs_children<E>(), mt[c]);
            EpiK<E>::template load<4, NM>(D, j, mt[c], in[c]);
          }
        }
        // ---- accumulators -> xs[slot][col][unit] (warp quadrant q holds TMEM lanes 32q..32q+31) ----
        pwait_warp(done, tcount & 1);
        if (D.trace && et == 0 && tr1 == 0) tr1 = gtime();
        ptx::tc_fence_after();
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)P.acc0;
#pragma unroll
        for (int s = 0; s < L::NSLOT; ++s) {
          constexpr int UG = L::UG;
          const int g = L::grp(s);
          if (q * 32 < g * UG || q * 32 >= (g + 1) * UG) continue;
          const int urow = q * 32 - g * UG + lane;
          for (int c0 = half * (nt / 2); c0 < (half + 1) * (nt / 2); c0 += 8) {
            float v[8];
            ptx::tmem_ld<8>(tq + L::acc(s, 0) * nt + c0, v);
#pragma unroll
            for (int a = 1; a < L::nacc(s); ++a) {
              float w8[8];
              ptx::tmem_ld<8>(tq + L::acc(s, a) * nt + c0, w8);
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] += w8[e];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) xs[(s * kPMaxNT + c0 + e) * UG + urow] = v[e];
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tmem_empty);
        ptx::named_bar_sync(1, 256);
        if (D.trace && et == 0 && tr3 == 0) tr3 = gtime();
        // ---- fused cell epilogue: thread -> (unit quad, columns) ----
#pragma unroll 1
        while (base < items) {
          FV<4> acc[CH][NE];
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int it = base + 256 * c;
            if (it >= items) continue;
            const int col = it / quads;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              float4 sum = *reinterpret_cast<const float4*>(xs + (L::e_slot(e, 0) * kPMaxNT + col) * L::UG + quad * 4);
#pragma unroll
              for (int z = 1; z < L::e_n(e); ++z) {
                const float4 x = *reinterpret_cast<const float4*>(
                    xs + (L::e_slot(e, z) * kPMaxNT + col) * L::UG + quad * 4);
                sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
              }
              acc[c][e].v[0] = sum.x; acc[c][e].v[1] = sum.y; acc[c][e].v[2] = sum.z; acc[c][e].v[3] = sum.w;
            }
          }
#pragma unroll
          for (int c = 0; c < CH; ++c)
            if (base + 256 * c < items) EpiK<E>::template store<__nv_bfloat16, 4, NM>(D, j, mt[c], acc[c], in[c], uc);
          base += 256 * CH;
#pragma unroll
          for (int c = 0; c < CH; ++c) {                 // next round (large tiles / FC): load, then loop
            const int it = base + 256 * c;
            if (it < items) {
              load_meta(D, p0 + it / quads, epi_needs_children<E>(), mt[c]);
              EpiK<E>::template load<4, NM>(D, j, mt[c], in[c]);
            }
          }
        }
        unsigned long long tl = 0;
        if (D.trace) { tl = gtime(); atomicMax(&s_tmax, tl); }
        ptx::named_bar_sync(1, 256);                     // xs free for the next tile
        if (D.trace && et == 0 && jt == 0) { ptrace(D, 6000 + E, blockIdx.x, i, tr3, tl, s_tmax, gtime(), 0); s_tmax = 0; }
      }
      if (i + 1 < nlev) {                                // task V_t complete cluster-wide before V_t+-1
        ptx::named_bar_sync(1, 256);
        if (et < 32) {
          if (D.trace && et == 0) tr2 = gtime();
          if (ntile > 0) {                               // cluster-uniform: same rows for every unit block
            if (et < P.nub) cluster_arrive(cbar, et);    // one warp instruction: all peers at once
            if (et == 0) cluster_wait(cbar, (uint32_t)(nbar & 1));
            ++nbar;
          }
          if (et == 0) {
            gate_set(gate, i + 1);
            if (D.trace) ptrace(D, 2000 + E, blockIdx.x, (unsigned long long)i | ((unsigned long long)M << 16), tr0, tr1,
                                tr2, gtime(), tr3);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kPMma) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  cluster_sync_all();                                 // no peer touches this CTA's barrier after exit
}

// =====================================================================================
// host side
// =====================================================================================
struct PersistState {
  CUtensorMap A_fwd[4], A_bwd[4];     // per row group (box 64 x UG)
  CUtensorMap B_hk[3], B_dz[3];       // 3D {64, NT, sk} boxes over Hk / dZ
  PPlan fwd{}, bwd{};
  PbwdState* kbwd = nullptr;          // Tree-LSTM backward: K-split kernel (persist_bwd.cu)
  std::string kbwd_why;
  int num_sms = 0;
};

static PFN_cuTensorMapEncodeTiled_v12000 p_encode = nullptr;

static bool enc2(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_elems,
                 uint32_t box_cols, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return p_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// [rows, width] row-major arena viewed as {64 k, row, k-block}: one box = sk stacked K-major
// SW128 tiles of NT rows (smem order [kb][row][64]).
static bool enc3(CUtensorMap* m, const void* base, uint64_t width, uint64_t rows, uint32_t nt, uint32_t sk) {
  cuuint64_t dims[3] = {64, rows, width / 64};
  cuuint64_t strides[2] = {width * 2, 128};
  cuuint32_t box[3] = {64, nt, sk};
  cuuint32_t es[3] = {1, 1, 1};
  return p_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static void plan_slot(PPlan& P, int grp, int nacc, const int* accs) {
  const int s = P.nslot++;
  P.slot_grp[s] = grp;
  P.slot_nacc[s] = nacc;
  for (int a = 0; a < nacc; ++a) P.slot_acc[s][a] = accs[a];
}
static void plan_e(PPlan& P, int n, const int* slots) {
  const int e = P.ne++;
  P.e_n[e] = n;
  for (int z = 0; z < n; ++z) P.e_slot[e][z] = slots[z];
}

// smem offsets, pipeline depth, TMEM budget; false if the plan does not fit one CTA.
// tsA: the weights are staged once through smem and copied into TMEM columns [0, 32 nkbA),
// the accumulators follow; the B stages then reuse the staging area.
static bool plan_layout(PPlan& P, bool tsA) {
  const int A = P.nkbA * kPKb;
  const int xs = P.nslot * kPMaxNT * P.UG * 4;
  const int avail = 232448 - 1024 - xs - 256 - 2 * kPMaxS * 8 - 64;
  // segments must be contiguous B columns (one box may span several)
  for (int sg = 1; sg < P.nseg; ++sg)
    if (P.seg_bcol[sg] != P.seg_bcol[0] + sg * P.nkbA * 64) return false;
  for (int sg = 0; sg < P.nseg; ++sg)
    if (P.seg_acc[sg] != sg) return false;           // the issue loop assumes accumulator sg for segment sg
  for (int sg = 0; sg < P.nseg; ++sg) {
    P.seg_init[sg] = 1;
    for (int e = 0; e < sg; ++e)
      if (P.seg_acc[e] == P.seg_acc[sg]) P.seg_init[sg] = 0;
  }
  // stage size: as few, large TMA boxes per tile as the pipeline admits -- one SM's boxes are serviced
  // one after another, ~1 us each (tools/trace_persist.py: a 5-box tile's last box lands 5.5 us after
  // its first, a 1-box tile's in one), so a 16-row tile is ONE box and larger tiles take few: up to
  // 2 x the 16-row tile (>= 64 KB), two stages at least, multiples of 16 KB (r02: cfg4 bwd levels
  // 0.258 -> 0.224 ms with the 80 KB Tree-LSTM backward box, fwd 0.185 -> 0.172 ms with 64 KB)
  const int tile16 = 16 * 128 * P.nseg * P.nkbA;
  int stage = std::min({avail / 2, std::max(tile16, 65536), 2 * tile16});
  stage = std::max(kPStageMin, stage / kPStageMin * kPStageMin);
  // A/B: B stage bytes (multiple of 16 KB), per pass / both passes
  if (const char* e = std::getenv(P.is_bwd ? "CAVS_PERSIST_STAGE_BWD" : "CAVS_PERSIST_STAGE_FWD")) {
    const int v = std::atoi(e);
    if (v >= kPStageMin && v <= 98304 && v % kPStageMin == 0) stage = v;
  } else if (const char* e2 = std::getenv("CAVS_PERSIST_STAGE")) {
    const int v = std::atoi(e2);
    if (v >= kPStageMin && v <= 98304 && v % kPStageMin == 0) stage = v;
  }
  P.tsA = tsA ? 1 : 0;
  int S;
  if (tsA) {
    S = std::min(kPMaxS, avail / stage);
    if (S * stage < A) return false;
    P.acc0 = P.nkbA * 32;
    P.xs_off = S * stage;
  } else {
    S = std::min(kPProd, (avail - A) / stage);
    P.acc0 = 0;
    P.xs_off = A + S * stage;
  }
  if (S < 2) return false;
  P.S = S;
  P.stage = stage;
  P.max_ni = -1;
  for (int i = 0; i < 3; ++i)
    if (P.acc0 + P.nacc * (16 << i) <= 512) P.max_ni = i;
  if (P.max_ni < 0) return false;
  P.meta_off = P.xs_off + xs;
  P.bar_off = (P.meta_off + 15) & ~15;
  // k-blocks per box (<= 256), never more than a tile has (a box past the arena's last k-block would be
  // zero-filled by the TMA: bytes moved for nothing)
  for (int i = 0; i < 3; ++i) P.sk[i] = std::min(stage / ((16 << i) * 128), P.nseg * P.nkbA);
  return true;
}
static int plan_smem(const PPlan& P) { return 1024 + P.bar_off + 2 * kPMaxS * 8 + 64; }

// smem attribute + how many clusters of nub CTAs (1 CTA per SM) can be resident at once
template <int E, int NE, int NM>
static int attr_and_clusters(int smem, int nub) {
  if (cudaFuncSetAttribute(k_persist<E, NE, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return 0;
  if (nub > 8 && cudaFuncSetAttribute(k_persist<E, NE, NM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nub * kMaxClusters, 1, 1);
  cfg.blockDim = dim3(kPThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nub; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_persist<E, NE, NM>, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

template <int E, int NE, int NM>
static void launch_p(const CUtensorMap* A, const CUtensorMap* B, const Dev& D, const PPlan& P, int t_first, int nlev,
                     int dir, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.nub * P.R, 1, 1);
  cfg.blockDim = dim3(kPThreads, 1, 1);
  cfg.dynamicSmemBytes = plan_smem(P);
  cfg.stream = s;
  // one cluster of nub unit-block CTAs per graph range; PDL: the weights stream in under the
  // previous kernel
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P.nub; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_persist<E, NE, NM>, A[0], A[1], A[2], A[3], B[0], B[1], B[2], D, P,
                                     t_first, nlev, dir);
  if (e != cudaSuccess) {                             // retry this launch without PDL
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_persist<E, NE, NM>, A[0], A[1], A[2], A[3], B[0], B[1], B[2], D, P, t_first, nlev, dir);
  }
}

PersistState* persist_init(const Dev& D, int max_vertices, std::string* why) {
  const char* env = std::getenv("CAVS_PERSIST");
  if (env && env[0] == '0') { *why = "disabled (CAVS_PERSIST=0)"; return nullptr; }
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int h = D.h, N = D.N;
  const int UG = lstm ? 32 : 64;
  if (h % 64 || h % UG || h / 64 > 8) { *why = "shape: needs h % 64 == 0 and h <= 512"; return nullptr; }
  if (!p_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      *why = "cuTensorMapEncodeTiled unavailable";
      return nullptr;
    }
    p_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  PersistState* ps = new PersistState();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&ps->num_sms, cudaDevAttrMultiProcessorCount, dev);
  const int nub = h / UG;
  if (nub > 16) { delete ps; *why = "more than 16 unit blocks (cluster size)"; return nullptr; }
  int R = kMaxClusters;                               // clusters (graph ranges), set from occupancy below
  const uint64_t Vp = (uint64_t)max_vertices + kPadRows;
  const int G = lstm ? 3 + N : 1;
  bool ok = true;
  PPlan F{}, B{};
  F.UG = B.UG = UG; F.nkbA = B.nkbA = h / 64; F.nub = B.nub = nub; F.R = B.R = R;
  if (lstm) {
    // forward: groups (i, o, u, f) of U4 [4h x h]; acc k = U4 . h_k (sum over k by linearity, Z11)
    F.ngrp = 4;
    for (int g = 0; g < 4; ++g) { F.grp_row0[g] = g * h; F.grp_col0[g] = 0; ok &= enc2(&ps->A_fwd[g], D.Wa, h, 4 * h, h, 64, UG); }
    F.nseg = N;
    for (int k = 0; k < N; ++k) { F.seg_bcol[k] = k * h; F.seg_acc[k] = k; }
    F.nacc = N;
    int all[4] = {0, 1, 2, 3};
    for (int g = 0; g < 3; ++g) plan_slot(F, g, N, all);
    for (int k = 0; k < N; ++k) plan_slot(F, 3, 1, &all[k]);
    for (int e = 0; e < 3 + N; ++e) plan_e(F, 1, &e);
    // backward: groups (U_i^T, U_o^T, U_u^T, U_f^T) rows of the output units; acc g = group g
    // against dz_g, acc 3+k = U_f^T group against dz_fk
    B.ngrp = 4;
    for (int g = 0; g < 3; ++g) { B.grp_row0[g] = 0; B.grp_col0[g] = g * h; ok &= enc2(&ps->A_bwd[g], D.Wc, 3 * h, h, 3 * h, 64, UG); }
    B.grp_row0[3] = 0; B.grp_col0[3] = 0; ok &= enc2(&ps->A_bwd[3], D.Wd, h, h, h, 64, UG);
    B.nseg = 3 + N;
    for (int g = 0; g < 3 + N; ++g) { B.seg_bcol[g] = g * h; B.seg_acc[g] = g; }
    B.nacc = 3 + N;
    for (int g = 0; g < 3; ++g) plan_slot(B, g, 1, &g);
    for (int k = 0; k < N; ++k) { const int a = 3 + k; plan_slot(B, 3, 1, &a); }
    const int iou[3] = {0, 1, 2};
    plan_e(B, 3, iou);
    for (int k = 0; k < N; ++k) { const int sl = 3 + k; plan_e(B, 1, &sl); }
  } else {
    // Tree-FC forward: groups (W_l, W_r) rows of the units = W_c [h x 2h] columns [0,h) / [h,2h)
    F.ngrp = 2;
    for (int g = 0; g < 2; ++g) { F.grp_row0[g] = 0; F.grp_col0[g] = g * h; ok &= enc2(&ps->A_fwd[g], D.Wa, 2 * h, h, 2 * h, 64, UG); }
    ps->A_fwd[2] = ps->A_fwd[3] = ps->A_fwd[0];
    F.nseg = 2; F.seg_bcol[0] = 0; F.seg_acc[0] = 0; F.seg_bcol[1] = h; F.seg_acc[1] = 1;
    F.nacc = 2;
    const int a0 = 0, a1 = 1;
    plan_slot(F, 0, 1, &a0); plan_slot(F, 1, 1, &a1);
    const int both[2] = {0, 1};
    plan_e(F, 2, both);
    // backward: groups (W_l^T, W_r^T) = WcT [2h x h] rows [0,h) / [h,2h) against dz
    B.ngrp = 2;
    for (int g = 0; g < 2; ++g) { B.grp_row0[g] = g * h; B.grp_col0[g] = 0; ok &= enc2(&ps->A_bwd[g], D.Wc, h, 2 * h, h, 64, UG); }
    ps->A_bwd[2] = ps->A_bwd[3] = ps->A_bwd[0];
    B.nseg = 1; B.seg_bcol[0] = 0; B.seg_acc[0] = 0;
    B.nacc = 1;
    plan_slot(B, 0, 1, &a0); plan_slot(B, 1, 1, &a0);
    plan_e(B, 1, &a0); plan_e(B, 1, &a1);
  }
  const char* ss = std::getenv("CAVS_PERSIST_SS");    // 1: weights in smem (SS MMA) instead of TMEM
  const bool tsA = !(ss && ss[0] == '1');
  B.is_bwd = 1;
  if (!plan_layout(F, tsA) || !plan_layout(B, tsA)) { delete ps; *why = "does not fit shared memory / TMEM"; return nullptr; }
  for (int i = 0; i < 3; ++i) {
    ok &= enc3(&ps->B_hk[i], D.Hk, (uint64_t)N * h, Vp, 16u << i, F.sk[i]);
    ok &= enc3(&ps->B_dz[i], D.dZ, (uint64_t)G * h, Vp, 16u << i, B.sk[i]);
  }
  if (!ok) { delete ps; *why = "tensor map encode failed"; return nullptr; }
  // clusters of nub CTAs, one CTA per SM (TMEM, shared memory); every cluster runs its own graph
  // range through all tasks, so only a cluster's own CTAs need to be co-resident
  int nc = kMaxClusters;
  auto occ = [&](int a, int b) { nc = std::min(nc, std::min(a, b)); };
  if (lstm) {
    switch (N) {
      case 1: attr_and_clusters<EPI_LSTM_FWD_INF, 4, 1>(plan_smem(F), nub); occ(attr_and_clusters<EPI_LSTM_FWD, 4, 1>(plan_smem(F), nub), attr_and_clusters<EPI_LSTM_BWD, 2, 1>(plan_smem(B), nub)); break;
      case 2: attr_and_clusters<EPI_LSTM_FWD_INF, 5, 2>(plan_smem(F), nub); occ(attr_and_clusters<EPI_LSTM_FWD, 5, 2>(plan_smem(F), nub), attr_and_clusters<EPI_LSTM_BWD, 3, 2>(plan_smem(B), nub)); break;
      case 3: attr_and_clusters<EPI_LSTM_FWD_INF, 6, 3>(plan_smem(F), nub); occ(attr_and_clusters<EPI_LSTM_FWD, 6, 3>(plan_smem(F), nub), attr_and_clusters<EPI_LSTM_BWD, 4, 3>(plan_smem(B), nub)); break;
      default: attr_and_clusters<EPI_LSTM_FWD_INF, 7, 4>(plan_smem(F), nub); occ(attr_and_clusters<EPI_LSTM_FWD, 7, 4>(plan_smem(F), nub), attr_and_clusters<EPI_LSTM_BWD, 5, 4>(plan_smem(B), nub)); break;
    }
  } else {
    attr_and_clusters<EPI_FC_FWD_INF, 1, 1>(plan_smem(F), nub);
    occ(attr_and_clusters<EPI_FC_FWD, 1, 1>(plan_smem(F), nub), attr_and_clusters<EPI_FC_BWD, 2, 1>(plan_smem(B), nub));
  }
  if (lstm) {                                          // the K-split backward shares the cluster table
    int kc = 0;
    ps->kbwd = pbwd_init(D, max_vertices, &kc, &ps->kbwd_why);
    if (ps->kbwd) nc = std::min(nc, kc);
  }
  const char* cenv = std::getenv("CAVS_PERSIST_CLUSTERS");    // debug / A-B: fewer clusters
  if (cenv && std::atoi(cenv) > 0) nc = std::min(nc, std::atoi(cenv));
  if (nc < 1) {
    if (ps->kbwd) pbwd_destroy(ps->kbwd);
    delete ps;
    *why = "no cluster of " + std::to_string(nub) + " CTAs fits";
    return nullptr;
  }
  F.R = B.R = R = nc;
  if (ps->kbwd) pbwd_set_clusters(ps->kbwd, nc);
  // opt-in (CAVS_PERSIST_MC=1): one multicast TMA per B box per cluster instead of one load per CTA.
  // Parity-tested, but measured 1-3 % slower at cfg2/3/4 (the per-task chain is latency-bound and
  // a multicast stage can be refilled only once all 16 CTAs freed it; profiles/r02_ablations.md)
  const char* mce = std::getenv("CAVS_PERSIST_MC");
  F.mc = B.mc = (mce && mce[0] == '1') ? 1 : 0;
  ps->fwd = F;
  ps->bwd = B;
  return ps;
}

void persist_destroy(PersistState* ps) {
  if (ps && ps->kbwd) pbwd_destroy(ps->kbwd);
  delete ps;
}

int persist_clusters(const PersistState* ps) { return ps ? ps->fwd.R : 0; }
bool persist_has_kbwd(const PersistState* ps) { return ps && ps->kbwd; }

static bool D_is_lstm(const PersistState* ps) { return ps->fwd.ngrp == 4; }

std::string persist_describe(const PersistState* ps) {
  const PPlan& F = ps->fwd;
  const PPlan& B = ps->bwd;
  return "persistent: grid " + std::to_string(F.nub * F.R) + " (units/CTA " + std::to_string(F.UG) + ", " +
         (F.mc ? "B boxes multicast per cluster, " : "") +
         std::to_string(F.R) + " clusters of " + std::to_string(F.nub) + " over graph ranges), weights in " + (F.tsA ? "TMEM" : "smem") + ", stages fwd " + std::to_string(F.S) +
         " bwd " + std::to_string(B.S) + ", max task tile fwd " + std::to_string(16 << F.max_ni) + " bwd " +
         std::to_string(16 << B.max_ni) +
         (ps->kbwd ? "; " + pbwd_describe(ps->kbwd)
                   : (D_is_lstm(ps) ? "; bwd gate-grouped (K-split unavailable: " + ps->kbwd_why + ")" : std::string()));
}

void persist_forward(const Dev& D, PersistState* ps, int T, cudaStream_t s) {
  if (T <= 1 && !D.sync_free) return;
  if (D.sync_free) T = 0;                             // launch args (1, T - 1) = (1, -1): tasks from the device
  const PPlan& P = ps->fwd;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    if (D.infer) {                                    // inference-only forward: no activations for dF
      switch (D.N) {
        case 1: launch_p<EPI_LSTM_FWD_INF, 4, 1>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
        case 2: launch_p<EPI_LSTM_FWD_INF, 5, 2>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
        case 3: launch_p<EPI_LSTM_FWD_INF, 6, 3>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
        default: launch_p<EPI_LSTM_FWD_INF, 7, 4>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
      }
      return;
    }
    switch (D.N) {
      case 1: launch_p<EPI_LSTM_FWD, 4, 1>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
      case 2: launch_p<EPI_LSTM_FWD, 5, 2>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
      case 3: launch_p<EPI_LSTM_FWD, 6, 3>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
      default: launch_p<EPI_LSTM_FWD, 7, 4>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s); break;
    }
  } else if (D.infer) {
    launch_p<EPI_FC_FWD_INF, 1, 1>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s);
  } else {
    launch_p<EPI_FC_FWD, 1, 1>(ps->A_fwd, ps->B_hk, D, P, 1, T - 1, 1, s);
  }
}

void persist_backward(const Dev& D, PersistState* ps, int T, cudaStream_t s) {
  if (T <= 1 && !D.sync_free) return;
  if (D.sync_free) T = 0;                             // launch args (T - 1, T - 1) = (-1, -1): from the device
  if (ps->kbwd) { pbwd_launch(D, ps->kbwd, T, s); return; }
  const PPlan& P = ps->bwd;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    switch (D.N) {
      case 1: launch_p<EPI_LSTM_BWD, 2, 1>(ps->A_bwd, ps->B_dz, D, P, T - 1, T - 1, -1, s); break;
      case 2: launch_p<EPI_LSTM_BWD, 3, 2>(ps->A_bwd, ps->B_dz, D, P, T - 1, T - 1, -1, s); break;
      case 3: launch_p<EPI_LSTM_BWD, 4, 3>(ps->A_bwd, ps->B_dz, D, P, T - 1, T - 1, -1, s); break;
      default: launch_p<EPI_LSTM_BWD, 5, 4>(ps->A_bwd, ps->B_dz, D, P, T - 1, T - 1, -1, s); break;
    }
  } else {
    launch_p<EPI_FC_BWD, 2, 1>(ps->A_bwd, ps->B_dz, D, P, T - 1, T - 1, -1, s);
  }
}

}  // namespace cavs
