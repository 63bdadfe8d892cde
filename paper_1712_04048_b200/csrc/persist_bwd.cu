// persist_bwd.cu — BF16 mode, Tree-LSTM: the persistent backward level kernel, K-split
// weight-stationary with a DSMEM reduction (Alg. 1 BACKWARD; gradients
// are added; gather's adjoint is scatter).
//
// Per parent vertex p of task V_t and child slot k the level contraction is
//     dh_k(p) = U_iou^T dz_iou(p) + U_f^T dz_fk(p)       (dz_iou = [dz_i | dz_o | dz_u])
// a sum over K = 3h + h weight rows per output unit j.  The forward kernel's decomposition (a CTA
// owns 32 units x 4 gates, persist.cu) would multiply every dz segment against all four 32-row
// gate groups and keep one group: 4x the tensor-core work.  Here every MMA row is an output unit:
//
//   cluster = nub unit blocks (128 output units each) x 4 K-slices (nub = h / 128, <= 16 CTAs);
//   CTA (ub, ks) keeps rows [128 ub, +128) of U_iou^T restricted to the iou k-blocks [i0, i1) and
//   of U_f^T restricted to [f0, f1) resident in TMEM (the slices are balanced: every CTA holds
//   ~3h/256 + h/256 k-blocks of 64);
//   per task tile (NT = 16/32/64 task rows) it accumulates acc_iou = U_iou^T[:, i0:i1] dz_iou and
//   acc_k = U_f^T[:, f0:f1] dz_fk[f0:f1] for every child slot k (A from TMEM, B = the task's
//   contiguous dZ rows by TMA);
//   the epilogue sends the partials P_k = acc_iou + acc_k of output units [32 q, +32) to CTA
//   (ub, q) of its unit block (st.async into q's receive buffer, completing bytes on q's
//   mbarrier); CTA (ub, ks) sums the four K-slices' partials in fixed order (deterministic) and
//   runs the fused child dF of cells.cuh on units [128 ub + 32 ks, +32).
//
// Tasks are separated by the cluster-local task barrier of persist_common.cuh (the graphs of a
// batch are independent: one cluster per graph range, table crow[t][r]).
//
//   warps 0-2: TMA producers (resident weights once, then B boxes {64 k, NT rows, kbb k-blocks}),
//   warp 3:    TMEM allocator + MMA issuer,
//   warps 4-11: partial exchange, fused dF epilogue, task barrier.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "persist.h"
#include "persist_common.cuh"

namespace cavs {

constexpr int kBThreads = 384;
constexpr int kBProd = 3;
constexpr int kBMma = 3;
constexpr int kBEpi0 = 4;
constexpr int kBKb = 16384;        // one resident weight k-block: 128 rows x 64 bf16 (SW128)
constexpr int kBMaxS = 16;
constexpr int kBKS = 4;            // K-slices per unit block

struct BPlan {
  int nub, R, csize;               // unit blocks, clusters, CTAs per cluster (= 4 nub)
  int h64;                         // h / 64
  int i0[kBKS], ni[kBKS];          // iou k-blocks of K-slice ks
  int f0[kBKS], nf[kBKS];          // U_f k-blocks of K-slice ks
  int kbb;                         // k-blocks per B box
  int S, stage;                    // pipeline stages, bytes per stage (one box at NT = 64)
  int acc0;                        // first accumulator column (after the resident weights)
  int max_ni;                      // largest task tile index (NT = 16 << ni)
  int rc;                          // receive-buffer columns (= max NT)
  int recv_off, bar_off;
};

__device__ __forceinline__ void st_async_b32(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
               ::"r"(raddr), "r"(__float_as_uint(v)), "r"(rbar) : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

// MMA issue of one tile: segment 0 = iou (A k-blocks [0, ni), accumulator 0), segment 1 + k =
// child slot k (A k-blocks [ni, ni + nf), accumulator 1 + k); one box = kbb k-blocks.
template <int NT, int NM>
__device__ __forceinline__ void bmma_tile(int ni, int nf, int kbb, int S, uint32_t stage16, uint32_t acc0,
                                          uint32_t b_lo, uint64_t* full, uint64_t* empty, int& step) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
#pragma unroll 1
  for (int sg = 0; sg < 1 + NM; ++sg) {
    const int nkb = sg == 0 ? ni : nf;
    const uint32_t abase = sg == 0 ? 0u : (uint32_t)ni * 32u;
    const uint32_t d = acc0 + (uint32_t)(sg * NT);
#pragma unroll 1
    for (int kb = 0; kb < nkb; kb += kbb, ++step) {
      const int s = step % S;
      pwait_warp(&full[s], (step / S) & 1);
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        uint32_t bl = b_lo + (uint32_t)s * stage16;
        for (int g = 0; g < kbb; ++g) {
          const uint32_t at = abase + (uint32_t)(kb + g) * 32u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_bf16_ts(d, at + kk * 8, sw128_desc(bl + kk * 2), idesc, (kb + g == 0 && kk == 0) ? 0u : 1u);
          bl += (NT * 128) >> 4;
        }
        ptx::mma_commit(&empty[s]);
      }
      __syncwarp();
    }
  }
}

template <int NM>
__global__ void __launch_bounds__(kBThreads, 1)
k_pbwd(const __grid_constant__ CUtensorMap ma_iou, const __grid_constant__ CUtensorMap ma_f,
       const __grid_constant__ CUtensorMap mb16, const __grid_constant__ CUtensorMap mb32,
       const __grid_constant__ CUtensorMap mb64, Dev D, BPlan P, int t_first, int nlev) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                          // weight staging, then B stages
  uint8_t* sB = smem;
  float* recv = reinterpret_cast<float*>(smem + P.recv_off);   // [4 src][NM][rc cols][32 units]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bar_off);
  uint64_t* empty = full + kBMaxS;
  uint64_t* done = empty + kBMaxS;
  uint64_t* tmem_empty = done + 1;
  uint64_t* abar = tmem_empty + 1;
  uint64_t* acopy = abar + 1;
  uint64_t* cbar = acopy + 1;                                  // cluster task barrier
  uint64_t* rfull = cbar + 1;                                  // partials of the 4 K-slices arrived
  uint64_t* rfree = rfull + 1;                                 // the 4 receivers consumed this CTA's partials
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfree + 1);
  int* gate = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = blockIdx.x % P.csize, r = blockIdx.x / P.csize;
  const int ub = rank / kBKS, ks = rank % kBKS;
  const int ni = P.ni[ks], nf = P.nf[ks], nA = ni + nf;
  const int S = P.S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::mbar_init(done, 1);
    ptx::mbar_init(tmem_empty, 8);
    ptx::mbar_init(abar, 1);
    ptx::mbar_init(acopy, 1);
    ptx::mbar_init(cbar, P.csize);
    ptx::mbar_init(rfull, 1);
    ptx::mbar_init(rfree, kBKS);
    *gate = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kBMma) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kBProd) {
    // ------------------------------------------------------------------ producers
    if (lane == 0) {
      const int w = warp;
      if (w == 0) {                                   // resident weights: nA k-blocks of 128 rows
        ptx::tma_prefetch(&ma_iou); ptx::tma_prefetch(&ma_f);
        ptx::mbar_arrive_expect_tx(abar, (uint32_t)nA * kBKb);
        for (int a = 0; a < nA; ++a) {
          if (a < ni) ptx::tma_load_2d(sA + a * kBKb, &ma_iou, (P.i0[ks] + a) * 64, ub * 128, abar);
          else ptx::tma_load_2d(sA + a * kBKb, &ma_f, (P.f0[ks] + a - ni) * 64, ub * 128, abar);
        }
      }
      ptx::tma_prefetch(&mb16); ptx::tma_prefetch(&mb32); ptx::tma_prefetch(&mb64);
      pwait(acopy, 0);                                // the stages overlay the weights' staging
      ptx::griddep_wait();
      const int seg_kb0[1 + kMaxN] = {P.i0[ks], 3 * P.h64 + P.f0[ks], 4 * P.h64 + P.f0[ks], 5 * P.h64 + P.f0[ks],
                                      6 * P.h64 + P.f0[ks]};
      int step = 0;
      for (int i = 0; i < nlev; ++i) {
        const int t = t_first - i;
        int lo, M;
        cl_rows(D, t, r, lo, M);
        const int nix = nt_index(M, 1, P.max_ni), nt = 16 << nix;
        const int ntile = (M + nt - 1) / nt;
        if (ntile == 0) continue;
        const CUtensorMap* mb = nix == 0 ? &mb16 : nix == 1 ? &mb32 : &mb64;
        const uint32_t bytes = (uint32_t)nt * 128u * (uint32_t)P.kbb;
        if (i > 0) {
          while (gate_get(gate) < i) { }              // task V_t+1 done cluster-wide (acquire)
          ptx::fence_proxy_async_global();            // its dZ writes -> this thread's TMA reads
        }
        if (D.trace && w == 0) ptrace(D, 7200, blockIdx.x, i, gtime(), 0, 0, 0, 0);
        for (int j = 0; j < ntile; ++j) {
          const int p0 = lo + j * nt;
          for (int sg = 0; sg < 1 + NM; ++sg) {
            const int nkb = sg == 0 ? ni : nf;
            for (int kb = 0; kb < nkb; kb += P.kbb, ++step) {
              const int s = step % S;
              if (s % kBProd != w) continue;
              if (step >= S) pwait(&empty[s], ((step / S) & 1) ^ 1);
              ptx::mbar_arrive_expect_tx(&full[s], bytes);
              ptx::tma_load_3d(sB + s * P.stage, mb, 0, p0, seg_kb0[sg] + kb, &full[s]);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kBMma) {
    // ------------------------------------------------------------------ MMA issuer
    if (tmem != 0) __trap();                          // alone on the SM: columns start at 0
    pwait_warp(abar, 0);
    ptx::tc_fence_after();
    if (ptx::elect_one()) {                           // weights -> TMEM columns [0, 32 nA)
      for (int a = 0; a < nA; ++a)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::tmem_cp_128x256b((uint32_t)(a * 32 + kk * 8),
                                sw128_desc(((ptx::smem_u32(sA + a * kBKb + kk * 32) >> 4) & 0x3FFF) | (1u << 16)));
      ptx::mma_commit(acopy);
    }
    __syncwarp();
    pwait_warp(acopy, 0);
    ptx::tc_fence_after();
    const uint32_t b_lo = ((ptx::smem_u32(sB) >> 4) & 0x3FFF) | (1u << 16);
    const uint32_t stage16 = (uint32_t)(P.stage >> 4), acc0 = (uint32_t)P.acc0;
    int step = 0, tcount = 0;
    for (int i = 0; i < nlev; ++i) {
      const int t = t_first - i;
      int lo, M;
      cl_rows(D, t, r, lo, M);
      const int nix = nt_index(M, 1, P.max_ni), nt = 16 << nix;
      const int ntile = (M + nt - 1) / nt;
      const unsigned long long tm0 = D.trace ? gtime() : 0;
      for (int j = 0; j < ntile; ++j, ++tcount) {
        if (tcount > 0) { pwait_warp(tmem_empty, (tcount - 1) & 1); ptx::tc_fence_after(); }
        if (nix == 0) bmma_tile<16, NM>(ni, nf, P.kbb, S, stage16, acc0, b_lo, full, empty, step);
        else if (nix == 1) bmma_tile<32, NM>(ni, nf, P.kbb, S, stage16, acc0, b_lo, full, empty, step);
        else bmma_tile<64, NM>(ni, nf, P.kbb, S, stage16, acc0, b_lo, full, empty, step);
        if (ptx::elect_one()) ptx::mma_commit(done);
        __syncwarp();
      }
      if (D.trace && ntile > 0 && lane == 0) ptrace(D, 7100, blockIdx.x, i, tm0, gtime(), nt, 0, 0);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ exchange + epilogue (8 warps)
    const int et = threadIdx.x - kBEpi0 * 32;         // 0..255
    const int q = warp & 3, half = (warp - kBEpi0) >> 2;
    const int quad = et & 7;                          // 8 unit quads of this CTA's 32 output units
    const int j = ub * 128 + ks * 32 + quad * 4;
    const int rc = P.rc;
    // q's receive buffer, slot of this K-slice, row `lane`; q's rfull barrier
    const uint32_t r_dst = mapa_u32(ptx::smem_u32(recv + ((size_t)ks * NM * rc) * 32 + lane), ub * kBKS + q);
    const uint32_t r_bar = mapa_u32(ptx::smem_u32(rfull), ub * kBKS + q);
    ptx::griddep_wait();
    const UnitC<4> uc{};
    int tcount = 0, nbar = 0;
    for (int i = 0; i < nlev; ++i) {
      const int t = t_first - i;
      int lo, M;
      cl_rows(D, t, r, lo, M);
      const int nix = nt_index(M, 1, P.max_ni), nt = 16 << nix;
      const int ntile = (M + nt - 1) / nt;
      if (i > 0 && ntile > 0) {
        if (lane == 0) while (gate_get(gate) < i) { }
        __syncwarp();
      }
      unsigned long long tr[6] = {0, 0, 0, 0, 0, 0};
      if (D.trace) tr[0] = gtime();
      for (int jt = 0; jt < ntile; ++jt, ++tcount) {
        const int p0 = lo + jt * nt;
        const int valid = min(nt, lo + M - p0);
        const int items = 8 * valid;
        // first round of (quad, column) items: metadata + cell inputs while the MMAs run
        VMeta mt;
        typename EpiK<EPI_LSTM_BWD>::template In<4, NM> in;
        int base = et;
        if (base < items) {
          load_meta(D, p0 + base / 8, true, mt);
          EpiK<EPI_LSTM_BWD>::template load<4, NM>(D, j, mt, in);
        }
        if (et == 0) ptx::mbar_arrive_expect_tx(rfull, (uint32_t)(kBKS * NM * nt * 32 * 4));
        pwait_warp(done, tcount & 1);
        ptx::tc_fence_after();
        if (D.trace && jt == 0) tr[1] = gtime();
        if (tcount > 0) pwait_warp(rfree, (tcount - 1) & 1);   // receivers consumed the last tile
        // ---- partials of output units [32 q, +32) -> CTA (ub, q): P_k = acc_iou + acc_k ----
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)P.acc0;
        for (int c0 = half * (nt / 2); c0 < (half + 1) * (nt / 2); c0 += 8) {
          float vi[8];
          ptx::tmem_ld<8>(tq + c0, vi);
#pragma unroll
          for (int k = 0; k < NM; ++k) {
            float v[8];
            if (nf > 0) {
              ptx::tmem_ld<8>(tq + (uint32_t)((1 + k) * nt) + c0, v);
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] += vi[e];
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = vi[e];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) st_async_b32(r_dst + (uint32_t)((k * rc + c0 + e) * 32 * 4), v[e], r_bar);
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tmem_empty);
        // ---- the four K-slices' partials of this CTA's units -> fused child dF ----
        if (D.trace && jt == 0) tr[2] = gtime();
        pwait_warp(rfull, tcount & 1);
        if (D.trace && jt == 0) tr[3] = gtime();
#pragma unroll 1
        while (base < items) {
          const int col = base / 8;
          FV<4> acc[1 + NM];
          acc[0] = zerov<4>();
#pragma unroll
          for (int k = 0; k < NM; ++k) {
            float4 sum = *reinterpret_cast<const float4*>(recv + ((size_t)(0 * NM + k) * rc + col) * 32 + quad * 4);
#pragma unroll
            for (int src = 1; src < kBKS; ++src) {
              const float4 x = *reinterpret_cast<const float4*>(recv + ((size_t)(src * NM + k) * rc + col) * 32 + quad * 4);
              sum.x += x.x; sum.y += x.y; sum.z += x.z; sum.w += x.w;
            }
            acc[1 + k].v[0] = sum.x; acc[1 + k].v[1] = sum.y; acc[1 + k].v[2] = sum.z; acc[1 + k].v[3] = sum.w;
          }
          EpiK<EPI_LSTM_BWD>::template store<__nv_bfloat16, 4, NM>(D, j, mt, acc, in, uc);
          base += 256;
          if (base < items) {
            load_meta(D, p0 + base / 8, true, mt);
            EpiK<EPI_LSTM_BWD>::template load<4, NM>(D, j, mt, in);
          }
        }
        ptx::named_bar_sync(1, 256);                  // recv consumed by every epilogue thread
        if (et < kBKS) cluster_arrive(rfree, ub * kBKS + et);   // release: the senders may overwrite
        if (D.trace) tr[4] = gtime();
      }
      if (i + 1 < nlev) {                             // V_t complete cluster-wide before V_t-1
        ptx::named_bar_sync(1, 256);
        if (et < 32) {
          if (ntile > 0) {
            if (et < P.csize) cluster_arrive(cbar, et);
            if (et == 0) cluster_wait(cbar, (uint32_t)(nbar & 1));
            ++nbar;
          }
          if (et == 0) gate_set(gate, i + 1);
        }
      }
      if (D.trace && et == 0 && ntile > 0)
      {
        ptrace(D, 7000, blockIdx.x, (unsigned long long)i | ((unsigned long long)M << 16), tr[0], tr[1], tr[2], tr[3],
               tr[4]);
        ptrace(D, 7001, blockIdx.x, i, gtime(), 0, 0, 0, 0);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kBMma) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  cluster_sync_all();                                 // no peer touches this CTA's smem after exit
}

// =====================================================================================
// host side
// =====================================================================================
struct PbwdState {
  CUtensorMap A_iou, A_f, B[3];
  BPlan P{};
};

static PFN_cuTensorMapEncodeTiled_v12000 b_encode = nullptr;

static bool benc2(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return b_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool benc3(CUtensorMap* m, const void* base, uint64_t width, uint64_t rows, uint32_t nt, uint32_t kbb) {
  cuuint64_t dims[3] = {64, rows, width / 64};
  cuuint64_t strides[2] = {width * 2, 128};
  cuuint32_t box[3] = {64, nt, kbb};
  cuuint32_t es[3] = {1, 1, 1};
  return b_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int pbwd_smem(const BPlan& P) { return 1024 + P.bar_off + (2 * kBMaxS + 8) * 8 + 64; }

template <int NM>
static int pbwd_attr_clusters(const BPlan& P) {
  const int smem = pbwd_smem(P);
  if (cudaFuncSetAttribute(k_pbwd<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
  if (P.csize > 8 && cudaFuncSetAttribute(k_pbwd<NM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.csize * kMaxClusters, 1, 1);
  cfg.blockDim = dim3(kBThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P.csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_pbwd<NM>, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

PbwdState* pbwd_init(const Dev& D, int max_vertices, int* clusters, std::string* why) {
  // Opt-in (CAVS_PBWD=1): measured on B200 at cfg4 it issues 4x fewer MMAs than the gate-grouped
  // backward but the per-tile DSMEM exchange costs more than the MMA issue it saves (bwd levels
  // 293 vs 252 us, profiles/r02_ablations.md), so the gate-grouped kernel stays the default.
  const char* env = std::getenv("CAVS_PBWD");
  if (!env || env[0] != '1') { *why = "off (opt-in: CAVS_PBWD=1)"; return nullptr; }
  const int h = D.h, N = D.N;
  if (D.cell != CAVS_CELL_TREE_LSTM || h % 128 || h < 128 || h > 512) {
    *why = "needs Tree-LSTM with h % 128 == 0, 128 <= h <= 512";
    return nullptr;
  }
  if (!b_encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn) {
      *why = "cuTensorMapEncodeTiled unavailable";
      return nullptr;
    }
    b_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  BPlan P{};
  P.h64 = h / 64;
  P.nub = h / 128;
  P.csize = P.nub * kBKS;
  const int n_i = 3 * P.h64, n_f = P.h64;
  int g = 0, nA_max = 0;
  for (int ks = 0; ks < kBKS; ++ks) {                 // balanced K-slices
    P.i0[ks] = ks * n_i / kBKS; P.ni[ks] = (ks + 1) * n_i / kBKS - P.i0[ks];
    P.f0[ks] = ks * n_f / kBKS; P.nf[ks] = (ks + 1) * n_f / kBKS - P.f0[ks];
    g = std::gcd(g, std::gcd(P.ni[ks], P.nf[ks]));
    nA_max = std::max(nA_max, P.ni[ks] + P.nf[ks]);
  }
  P.kbb = std::max(1, std::min(g, 2));                // boxes of <= 2 k-blocks (16 KB at NT = 64)
  if (g % P.kbb) P.kbb = 1;
  P.acc0 = nA_max * 32;
  P.stage = P.kbb * 64 * 128;
  const int smem_total = 232448 - 1024 - (2 * kBMaxS + 8) * 8 - 64 - 64;
  P.max_ni = -1;
  const char* mx = std::getenv("CAVS_PBWD_MAXNT");     // A/B: cap the task tile (16 / 32 / 64)
  const int ix_cap = mx ? (std::atoi(mx) <= 16 ? 0 : std::atoi(mx) <= 32 ? 1 : 2) : 2;
  for (int ix = ix_cap; ix >= 0 && P.max_ni < 0; --ix) {
    const int nt = 16 << ix;
    if (P.acc0 + (1 + N) * nt > 512) continue;
    const int recv = kBKS * N * nt * 32 * 4;
    const int avail = smem_total - recv;
    const int S = std::min(kBMaxS, avail / P.stage);
    if (S < 2 || S * P.stage < nA_max * kBKb) continue;
    P.max_ni = ix;
    P.rc = nt;
    P.S = S;
    P.recv_off = S * P.stage;
    P.bar_off = (P.recv_off + recv + 15) & ~15;
  }
  if (P.max_ni < 0) { *why = "does not fit shared memory / TMEM"; return nullptr; }
  PbwdState* st = new PbwdState();
  const uint64_t Vp = (uint64_t)max_vertices + kPadRows;
  bool ok = benc2(&st->A_iou, D.Wc, 3 * h, h, 128) && benc2(&st->A_f, D.Wd, h, h, 128);
  for (int i = 0; i < 3; ++i) ok &= benc3(&st->B[i], D.dZ, (uint64_t)(3 + N) * h, Vp, 16u << i, P.kbb);
  if (!ok) { delete st; *why = "tensor map encode failed"; return nullptr; }
  int nc = 0;
  switch (N) {
    case 1: nc = pbwd_attr_clusters<1>(P); break;
    case 2: nc = pbwd_attr_clusters<2>(P); break;
    case 3: nc = pbwd_attr_clusters<3>(P); break;
    default: nc = pbwd_attr_clusters<4>(P); break;
  }
  if (nc < 1) { delete st; *why = "no cluster of " + std::to_string(P.csize) + " CTAs fits"; return nullptr; }
  *clusters = std::min(nc, kMaxClusters);
  st->P = P;
  return st;
}

void pbwd_set_clusters(PbwdState* st, int R) { st->P.R = R; }
void pbwd_destroy(PbwdState* st) { delete st; }

std::string pbwd_describe(const PbwdState* st) {
  const BPlan& P = st->P;
  return "bwd K-split: clusters of " + std::to_string(P.csize) + " (" + std::to_string(P.nub) +
         " unit blocks x 4 K-slices, " + std::to_string(P.ni[0] + P.nf[0]) + " weight k-blocks/CTA), stages " +
         std::to_string(P.S) + ", max task tile " + std::to_string(16 << P.max_ni);
}

template <int NM>
static void pbwd_launch_n(const PbwdState* st, const Dev& D, int T, cudaStream_t s) {
  const BPlan& P = st->P;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.csize * P.R, 1, 1);
  cfg.blockDim = dim3(kBThreads, 1, 1);
  cfg.dynamicSmemBytes = pbwd_smem(P);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P.csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, k_pbwd<NM>, st->A_iou, st->A_f, st->B[0], st->B[1], st->B[2], D, P, T - 1, T - 1) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_pbwd<NM>, st->A_iou, st->A_f, st->B[0], st->B[1], st->B[2], D, P, T - 1, T - 1);
  }
}

void pbwd_launch(const Dev& D, const PbwdState* st, int T, cudaStream_t s) {
  if (T <= 1) return;
  switch (D.N) {
    case 1: pbwd_launch_n<1>(st, D, T, s); break;
    case 2: pbwd_launch_n<2>(st, D, T, s); break;
    case 3: pbwd_launch_n<3>(st, D, T, s); break;
    default: pbwd_launch_n<4>(st, D, T, s); break;
  }
}

}  // namespace cavs
