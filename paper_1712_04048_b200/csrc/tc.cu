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
  int nB; int b_col[3];      // B column bases in the arena
  int sum;                   // C = sum of the nB B tiles (child-sum h~)
  int nk;                    // k-blocks
  int nmma; int mma_a[6], mma_b[6], mma_acc[6];   // mma_b: 0..2 B tile, 3 = C
};
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
            const uint32_t bb = b.mma_b[m] == 3 ? st + P.offC : st + P.offB + b.mma_b[m] * B_TILE;
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

// =====================================================================================
// host side
// =====================================================================================
struct TcState {
  // K-major A (weights, box 64 x 128), K-major B (arenas, box 64 x NT), MN-major (box 64 x 64)
  CUtensorMap A[5];
  CUtensorMap B_hk, B_xp, B_dz;
  CUtensorMap M_dz, M_hs, M_hk, M_xp;
  bool use_simt = false;
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
    launch_I<EPI_LSTM_XPROJ, 4>(t, t->A[1], t->A[1], t->B_xp, D, X, 0, D.V, h, s); P.count(1);
    P.mark(CAVS_PH_FWD_LEVELS, s);
    // levels t >= 1: A = U4, B = child slots of the task's rows; h~ formed in smem
    PlanI F{};
    F.nb = 1;
    Bundle& f = F.b[0];
    f.map_a = 0; f.nA = 4; for (int g = 0; g < 4; ++g) f.a_row[g] = g * h; f.a_col0 = 0;
    f.nB = N; for (int k = 0; k < N; ++k) f.b_col[k] = k * h;
    f.sum = N >= 2; f.nk = h / BK;
    f.nmma = 3 + N;
    for (int g = 0; g < 3; ++g) { f.mma_a[g] = g; f.mma_b[g] = N >= 2 ? 3 : 0; f.mma_acc[g] = g; }
    for (int k = 0; k < N; ++k) { f.mma_a[3 + k] = 3; f.mma_b[3 + k] = k; f.mma_acc[3 + k] = 3 + k; }
    const SegListI Fs = fwd_segments(D);
    for (int tt = 1; tt < T; ++tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_FWD, Fs, lp[tt], lp[tt + 1], h, s);
      else if (N == 1) launch_I<EPI_LSTM_FWD, 4>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      else if (N == 2) launch_I<EPI_LSTM_FWD, 5>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      else if (N == 3) launch_I<EPI_LSTM_FWD, 6>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      else launch_I<EPI_LSTM_FWD, 7>(t, t->A[0], t->A[0], t->B_hk, D, F, lp[tt], lp[tt + 1], h, s);
      P.count(1);
    }
  } else {
    PlanI X{};
    X.nb = 1;
    X.b[0] = one(0, 0, 0, 0, d / BK, 0);
    launch_I<EPI_FC_XPROJ, 1>(t, t->A[1], t->A[1], t->B_xp, D, X, 0, D.V, h, s); P.count(1);
    P.mark(CAVS_PH_FWD_LEVELS, s);
    PlanI F{};
    F.nb = 1;
    F.b[0] = one(0, 0, 0, 0, 2 * h / BK, 0);
    const SegListI Fs = fwd_segments(D);
    for (int tt = 1; tt < T; ++tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_FWD, Fs, lp[tt], lp[tt + 1], h, s);
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
    for (int tt = T - 1; tt >= 1; --tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_LSTM_BWD, Bs, lp[tt], lp[tt + 1], h, s);
      else if (N == 1) launch_I<EPI_LSTM_BWD, 2>(t, t->A[2], t->A[3], t->B_dz, D, B, lp[tt], lp[tt + 1], h, s);
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
    for (int tt = T - 1; tt >= 1; --tt) {
      if (lp[tt + 1] - lp[tt] <= skmax) skinny_typeI<__nv_bfloat16>(D, EPI_FC_BWD, Bs, lp[tt], lp[tt + 1], h, s);
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
      launch_I<EPI_DX, 1>(t, t->A[4], t->A[4], t->B_dz, D, X, 0, V, d, s); P.count(1);
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
      launch_I<EPI_DX, 1>(t, t->A[4], t->A[4], t->B_dz, D, X, 0, V, d, s); P.count(1);
    }
  }
}

}  // namespace cavs
