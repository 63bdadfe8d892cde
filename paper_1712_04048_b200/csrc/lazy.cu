// lazy.cu — BF16 mode: the lazily batched parameter gradients (§3.5 "Lazy batching",
// the weight gradients of every task are summed once, after the backward loop) as ONE
// stream-K tcgen05 launch.
//
//   out[m, n] = sum_seg sum_{p in rows} A[p, a_col(seg) + m] * B[p, b_col(seg) + n]
//
// with A = dZ (gate pre-activation gradients) and B = the gather arena Hk (dU, by linearity of
// h~ = sum_k h_k) or the pulled inputs Xp (dW), both position-ordered arenas read MN-major
// straight from HBM/L2 (3-D TMA boxes {64 cols, 64 rows, chunks}, SWIZZLE_128B).  Jobs
// (Tree-LSTM: dU_iou, dU_f, dW_iou, dW_f; Tree-FC: dW_c, dW_x) are cut into 128 x 256 output
// tiles; all (tile, k-block) work of all jobs is laid end to end and split into equal contiguous
// ranges, one per CTA (stream-K), so every SM gets the same number of k-blocks regardless of
// the jobs' different depths.  A tile cut by a range boundary is finished by its pieces' CTAs:
// each writes its fp32 partial to a scratch slot, the last to arrive (per-tile counter) sums
// the slots in piece order (deterministic) and writes the packed dparams block; a tile in one
// piece goes straight to dparams.  K-blocks of dW without any pull record are skipped (the
// active list is built per CTA from k_pull's 64-row flags; the host plan's estimate is mapped
// proportionally onto the device count, so the pieces still tile the job exactly).
//
// 128 x 256 tiles (48 KB of operands per 64-deep k-block, 87 FLOP/B) instead of 128 x 128
// (64 FLOP/B): the k-loop streams from L2, whose throughput bounds the old split-K kernel.
//   warp 0: TMA producer, warp 1: TMEM allocator + MMA issuer (two 256-column accumulators, so
//   the epilogue of one piece overlaps the next piece's k-loop), warps 2-5: epilogue.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <queue>
#include <vector>

#include "lazy.h"
#include "ptx.cuh"

namespace cavs {

constexpr int kLThreads = 288;            // warps 0-3 TMA (one per stage), 4 MMA, 5-8 epilogue
constexpr int kLMma = 4, kLEpi0 = 5;
constexpr int kLBM = 128, kLBN = 256;      // output tile
constexpr int kLA = kLBM * 128;            // A stage: 128 MN x 64 K bf16 = 16 KB
constexpr int kLB = kLBN * 128;            // B stage: 256 MN x 64 K = 32 KB
constexpr int kLStage = kLA + kLB;
constexpr int kLS = 4;                     // pipeline stages
constexpr int kLPitch = 36;                // epilogue transpose pitch (floats)
constexpr int kLMaxItems = 640;
constexpr int kLMaxCta = 148;
constexpr int kLMaxAct = 2048;             // 64-row blocks of the active list (V <= 131k)
constexpr int kLSlot = kLBM * kLBN;        // floats per partial slot
constexpr int kLMinPiece = 8;              // k-blocks per CTA at least

struct LJob {
  int nseg, a_col[4], b_col[4];
  int k_lo, k_hi;        // position rows
  int skip;              // 1: only 64-row blocks with a pull record (rows [0, V))
  int bsrc;              // 0: Hk, 1: Xp
  int M, Ncols, ntn;     // output rows / cols, tiles along N
  int ld;                // dparams row pitch of the block
  long long out;         // dparams offset of the block
  int hblk, rowmap[4];   // internal row m -> packed row rowmap[m / hblk] + m % hblk
  int nkb;               // k-blocks per segment in the host plan (estimate for skip jobs)
  int dev_lo;            // 1 (sync-free mode): k_lo = level_ptr[1] read on the device, nkb an estimate
};
struct LItem {
  unsigned short gtile, ltile;   // tile id (counter index) / job-local tile
  unsigned char job, piece, npiece, pad;
  unsigned short slot;           // scratch slot of piece 0 (+piece); unused when npiece == 1
  int g0, g1;                    // job k-block range, host-plan units
};
struct LPlan {
  int nitems;
  LJob job[4];
  unsigned short cta_start[kLMaxCta + 1];
  LItem item[kLMaxItems];
};

__device__ __forceinline__ void lwait(uint64_t* bar, uint32_t parity) {
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

// actual k-block range [a, b) of an item and k-blocks per segment; the host plan's estimate is
// mapped proportionally onto the device count (pull-record blocks; internal rows in sync-free mode)
__device__ __forceinline__ void item_range(const LJob& J, const LItem& it, int n_act, int nkb_in, int& a, int& b,
                                           int& kps) {
  if (J.skip || J.dev_lo) {
    kps = J.skip ? n_act : nkb_in;
    const long long est = (long long)J.nseg * J.nkb, act = (long long)J.nseg * kps;
    a = est ? (int)((long long)it.g0 * act / est) : 0;
    b = est ? (int)((long long)it.g1 * act / est) : 0;
  } else {
    kps = J.nkb;
    a = it.g0;
    b = it.g1;
  }
}

__device__ __forceinline__ uint64_t mn_desc(uint32_t saddr) {   // MN-major SW128: LBO 8 KB (64-wide chunks), SBO 1 KB
  return ptx::sdesc_sw128(saddr, 8192, 1024);
}

__global__ void __launch_bounds__(kLThreads, 1)
k_lazy(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mHk,
       const __grid_constant__ CUtensorMap mXp, Dev D, const __grid_constant__ LPlan P) {
  extern __shared__ __align__(16) uint8_t l_raw[];
  uint8_t* smem = l_raw + ((1024u - (ptx::smem_u32(l_raw) & 1023u)) & 1023u);
  float* xs = reinterpret_cast<float*>(smem + kLS * kLStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(xs + 4 * 32 * kLPitch);
  uint64_t* empty = full + kLS;
  uint64_t* accf = empty + kLS;      // [2] accumulator ready
  uint64_t* acce = accf + 2;         // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);             // [0] n_act, [1] last arrival
  unsigned short* s_act = reinterpret_cast<unsigned short*>(s_flag + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = P.cta_start[blockIdx.x];
  int i1 = P.cta_start[blockIdx.x + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLS; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&accf[b], 1); ptx::mbar_init(&acce[b], 128); }
    ptx::fence_mbar_init();
  }
  if (warp == kLMma) ptx::tmem_alloc<512>(tmem_slot);
  bool need_act = false;
  for (int i = i0; i < i1; ++i) need_act |= P.job[P.item[i].job].skip != 0;
  ptx::griddep_wait();                                   // dZ of the backward pass, k_pull's flags
  if (dev_skip(D)) i1 = i0;                              // sync-free mode: invalid / DAG batch, no work
  const int lp1d = dev_lp1(D);                           // internal rows [lp1d, V) (dU jobs)
  const int nkb_in = lp1d < D.V ? cdiv(D.V - lp1d, 64) : 0;
  if (warp == 0) {
    int n = 0;
    if (need_act) {                                      // ascending list of 64-row blocks with a pull record
      const int nt = cdiv(D.V, 64);
      for (int b0 = 0; b0 < nt; b0 += 32) {
        const int f = (b0 + lane < nt) ? D.tile_x[b0 + lane] : 0;
        const unsigned m = __ballot_sync(~0u, f != 0);
        if (f) s_act[n + __popc(m & ((1u << lane) - 1u))] = (unsigned short)(b0 + lane);
        n += __popc(m);
      }
    }
    if (lane == 0) s_flag[0] = n;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_act = s_flag[0];

  if (warp < kLS) {
    // ---- TMA producers: warp w fills stage w (a single issuing thread serialises its boxes),
    //      lane 0 the A box (16 KB), lanes 1-2 the two halves of the B box (16 KB each) ----
    if (lane < 3) {
      if (warp == 0 && lane == 0) { ptx::tma_prefetch(&mA); ptx::tma_prefetch(&mHk); ptx::tma_prefetch(&mXp); }
      int step = 0;
      for (int i = i0; i < i1; ++i) {
        const LItem& it = P.item[i];
        const LJob& J = P.job[it.job];
        const int tm = it.ltile / J.ntn, tn = it.ltile % J.ntn;
        const CUtensorMap* mB = J.bsrc ? &mXp : &mHk;
        int a, b, kps;
        item_range(J, it, n_act, nkb_in, a, b, kps);
        for (int g = a; g < b; ++g, ++step) {
          const int s = step % kLS;
          if (s != warp) continue;
          const int seg = g / kps, j = g - seg * kps;
          const int r0 = J.skip ? 64 * (int)s_act[j] : (J.dev_lo ? lp1d : J.k_lo) + 64 * j;
          if (step >= kLS) lwait(&empty[s], ((step / kLS) & 1) ^ 1);
          uint8_t* st = smem + s * kLStage;
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&full[s], kLStage);
            ptx::tma_load_3d(st, &mA, 0, r0, (J.a_col[seg] + tm * kLBM) >> 6, &full[s]);
          } else {
            const int hb = lane - 1;
            ptx::tma_load_3d(st + kLA + hb * (kLB / 2), mB, 0, r0, ((J.b_col[seg] + tn * kLBN) >> 6) + 2 * hb, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kLMma) {
    // ---- MMA issuer: D[128 x 256] (+)= A^T B over the piece's k-blocks ----
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(kLBM, kLBN, 1, 1);
      int step = 0;
      for (int i = i0, k = 0; i < i1; ++i, ++k) {
        const LItem& it = P.item[i];
        const LJob& J = P.job[it.job];
        int a, b, kps;
        item_range(J, it, n_act, nkb_in, a, b, kps);
        const int buf = k & 1;
        if (k >= 2) lwait(&acce[buf], ((k - 2) >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * kLBN);
        for (int g = a; g < b; ++g, ++step) {
          const int s = step % kLS;
          lwait(&full[s], (step / kLS) & 1);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + s * kLStage), sb = sa + kLA;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_bf16(d, mn_desc(sa + kk * 2048), mn_desc(sb + kk * 2048), idesc, (g > a || kk > 0) ? 1u : 0u);
          ptx::mma_commit(&empty[s]);
        }
        ptx::mma_commit(&accf[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: thread = accumulator row (TMEM lane); 32 x 32 blocks transposed through smem
    //      so each store is a coalesced run of an output row ----
    const int q = warp & 3;
    const int et = threadIdx.x - 32 * kLEpi0;
    float* xw = xs + (warp - kLEpi0) * 32 * kLPitch;
    for (int i = i0, k = 0; i < i1; ++i, ++k) {
      const LItem& it = P.item[i];
      const LJob& J = P.job[it.job];
      const int tm = it.ltile / J.ntn, tn = it.ltile % J.ntn;
      int a, b, kps;
      item_range(J, it, n_act, nkb_in, a, b, kps);
      const int buf = k & 1;
      lwait(&accf[buf], (k >> 1) & 1);
      ptx::tc_fence_after();
      const bool direct = it.npiece == 1;
      const int mw = tm * kLBM + q * 32;                 // job row of this warp's first lane
      float* slot = D.lazy + (size_t)(it.slot + it.piece) * kLSlot;
      for (int cc = 0; cc < kLBN / 32; ++cc) {
        const int nc = tn * kLBN + cc * 32;
        if (nc >= J.Ncols) break;
        float v[32];
        if (b > a) {
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kLBN + cc * 32);
          ptx::tmem_ld16(ta, v);
          ptx::tmem_ld16(ta + 16, v + 16);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4*>(xw + lane * kLPitch + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        __syncwarp();
#pragma unroll
        for (int r4 = 0; r4 < 8; ++r4) {
          const int rr = r4 * 4 + (lane >> 3), c4 = (lane & 7) * 4;
          const int m = mw + rr, n = nc + c4;
          if (m < J.M && n < J.Ncols) {
            const float4 x = *reinterpret_cast<const float4*>(xw + rr * kLPitch + c4);
            float* dst = direct ? D.dparams + J.out + (size_t)(J.rowmap[m / J.hblk] + m % J.hblk) * J.ld + n
                                : slot + (size_t)(q * 32 + rr) * kLBN + cc * 32 + c4;
            *reinterpret_cast<float4*>(dst) = x;
          }
        }
        __syncwarp();
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&acce[buf]);
      if (!direct) {
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (et == 0) s_flag[1] = atomicAdd(D.tile_cnt + it.gtile, 1) == it.npiece - 1;
        ptx::named_bar_sync(1, 128);
        if (s_flag[1]) {                                 // last piece: sum the slots in piece order
          __threadfence();
          const float* base = D.lazy + (size_t)it.slot * kLSlot;
          // 8 rows x 2 float4 per lane in flight per slot (the reduction is the kernel's tail)
#pragma unroll 1
          for (int r8 = 0; r8 < 32; r8 += 8) {
            float4 acc[8][2];
#pragma unroll
            for (int rr = 0; rr < 8; ++rr)
#pragma unroll
              for (int hf = 0; hf < 2; ++hf)
                acc[rr][hf] = __ldcg(reinterpret_cast<const float4*>(base + (size_t)(q * 32 + r8 + rr) * kLBN + hf * 128 + lane * 4));
            for (int p = 1; p < it.npiece; ++p) {
              const float* sp = base + (size_t)p * kLSlot;
#pragma unroll
              for (int rr = 0; rr < 8; ++rr)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                  const float4 x = __ldcg(reinterpret_cast<const float4*>(sp + (size_t)(q * 32 + r8 + rr) * kLBN + hf * 128 + lane * 4));
                  acc[rr][hf].x += x.x; acc[rr][hf].y += x.y; acc[rr][hf].z += x.z; acc[rr][hf].w += x.w;
                }
            }
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
              const int m = tm * kLBM + q * 32 + r8 + rr;
              if (m < J.M) {
                float* orow = D.dparams + J.out + (size_t)(J.rowmap[m / J.hblk] + m % J.hblk) * J.ld;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                  const int n = tn * kLBN + hf * 128 + lane * 4;
                  if (n < J.Ncols) *reinterpret_cast<float4*>(orow + n) = acc[rr][hf];
                }
              }
            }
          }
          if (et == 0) D.tile_cnt[it.gtile] = 0;         // replayable
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kLMma) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// =====================================================================================
// host side
// =====================================================================================
struct LazyState {
  CUtensorMap A_dz, B_hk, B_xp;
  size_t slots = 0;               // scratch slots available in D.lazy
  int max_act = 0;
  LPlan plan{};                   // host staging of the kernel parameter (per context: thread-safe across contexts)
};

static PFN_cuTensorMapEncodeTiled_v12000 l_enc = nullptr;
static constexpr int kLSmem = 1024 + kLS * kLStage + 4 * 32 * kLPitch * 4 + (2 * kLS + 4) * 8 + 32 + 2 * kLMaxAct;

// [rows, width] bf16 arena viewed as {64 cols, rows, width / 64 chunks}: box {64, 64, chunks}
static bool lenc(CUtensorMap* m, const void* base, uint64_t width, uint64_t rows, uint32_t chunks) {
  cuuint64_t dims[3] = {64, rows, width / 64};
  cuuint64_t strides[2] = {width * 2, 128};
  cuuint32_t box[3] = {64, 64, chunks};
  cuuint32_t es[3] = {1, 1, 1};
  return l_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

LazyState* lazy_init(const Dev& D, int max_vertices) {
  const char* env = std::getenv("CAVS_LAZY");
  if (env && env[0] == '0') return nullptr;
  if (D.h % 64 || D.d % 64) return nullptr;
  const int Vp = max_vertices + kPadRows;
  if (cdiv(Vp, 64) > kLMaxAct) return nullptr;
  if (!l_enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return nullptr;
    l_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const uint64_t h = D.h, d = D.d, G = lstm ? 3 + D.N : 1;
  LazyState* l = new LazyState();
  bool ok = lenc(&l->A_dz, D.dZ, G * h, Vp, kLBM / 64) && lenc(&l->B_hk, D.Hk, (uint64_t)D.N * h, Vp, kLBN / 128) &&
            lenc(&l->B_xp, D.Xp, d, Vp, kLBN / 128);   // B: two half boxes per stage
  ok = ok && cudaFuncSetAttribute(k_lazy, cudaFuncAttributeMaxDynamicSharedMemorySize, kLSmem) == cudaSuccess;
  if (!ok) { delete l; return nullptr; }
  l->slots = lazy_floats(D) / kLSlot;
  return l;
}

void lazy_destroy(LazyState* l) { delete l; }

static LJob job(int nseg, const int* a_col, const int* b_col, int k_lo, int k_hi, int skip, int bsrc, int M, int Ncols,
                int ld, long long out, int hblk, const int* rowmap, int nkb) {
  LJob J{};
  J.nseg = nseg;
  for (int s = 0; s < nseg; ++s) { J.a_col[s] = a_col[s]; J.b_col[s] = b_col[s]; }
  J.k_lo = k_lo; J.k_hi = k_hi; J.skip = skip; J.bsrc = bsrc;
  J.M = M; J.Ncols = Ncols; J.ntn = cdiv(Ncols, kLBN);
  J.ld = ld; J.out = out; J.hblk = hblk;
  for (int g = 0; g < 4; ++g) J.rowmap[g] = rowmap[std::min(g, 3)];
  J.nkb = nkb;
  return J;
}
static LJob dev_rows(LJob J, bool on) {              // sync-free mode: internal rows from the device
  J.dev_lo = (on && !J.skip) ? 1 : 0;
  return J;
}

bool lazy_grads(const Dev& D, LazyState* l, cudaStream_t s) {
  if (!l || !D.dparams || (reinterpret_cast<uintptr_t>(D.dparams) & 15)) return false;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int h = D.h, d = D.d, N = D.N, V = D.V, lp1 = D.sync_free ? 0 : D.lp1;
  // internal rows [lp1, V); sync-free mode: level_ptr[1] is read on the device, the plan assumes
  // every row (the device maps it onto the actual count, item_range)
  const int nkb_in = lp1 < V ? cdiv(V - lp1, 64) : 0;
  // dW rows: the 64-row blocks holding a pull record; the plan assumes they are packed (trees:
  // the leaves [0, lp1); chains: every row); the device maps the plan onto the actual count
  const int nkb_x = std::min(cdiv(V, 64), cdiv(std::max(D.n_x, 0), 64));
  LPlan& P = l->plan;                                                      // host staging (kernel parameter), per context
  int nj = 0;
  const int zero4[4] = {0, 0, 0, 0};
  if (lstm) {
    const long long nW = 4LL * h * d, nU = 3LL * h * h;
    int bk[4], af[4], ident[4] = {0, 0, 0, 0}, iou[4] = {0, 2 * h, 3 * h, 3 * h};
    for (int k = 0; k < N; ++k) { bk[k] = k * h; af[k] = (3 + k) * h; }
    P.job[nj++] = dev_rows(job(N, zero4, bk, lp1, V, 0, 0, 3 * h, h, h, nW, 3 * h, ident, nkb_in), D.sync_free);  // dU_iou
    P.job[nj++] = dev_rows(job(N, af, bk, lp1, V, 0, 0, h, h, h, nW + nU, h, ident, nkb_in), D.sync_free);        // dU_f
    P.job[nj++] = job(1, zero4, zero4, 0, V, 1, 1, 3 * h, d, d, 0, h, iou, nkb_x);               // dW_i,o,u
    P.job[nj++] = job(N, af, zero4, 0, V, 1, 1, h, d, d, (long long)h * d, h, ident, nkb_x);     // dW_f
  } else {
    P.job[nj++] = dev_rows(job(1, zero4, zero4, lp1, V, 0, 0, h, 2 * h, 2 * h, 0, h, zero4, nkb_in), D.sync_free);  // dW_c
    P.job[nj++] = job(1, zero4, zero4, 0, V, 1, 1, h, d, d, 2LL * h * h, h, zero4, nkb_x);       // dW_x
  }
  // stream-K partition of the (tile, k-block) work
  struct T { int job, ltile; long long w; };
  std::vector<T> tiles;
  long long W = 0;
  for (int j = 0; j < nj; ++j) {                       // tm fastest: CTAs of one wave share B column blocks
    const LJob& J = P.job[j];
    const int ntm = cdiv(J.M, kLBM);
    for (int tn = 0; tn < J.ntn; ++tn)
      for (int tm = 0; tm < ntm; ++tm) {
        tiles.push_back({j, tm * J.ntn + tn, (long long)J.nseg * J.nkb});
        W += (long long)J.nseg * J.nkb;
      }
  }
  if ((int)tiles.size() > kLazyMaxTiles) return false;
  const int grid = (int)std::max<long long>(1, std::min<long long>(kLMaxCta, W / kLMinPiece));
  std::vector<std::vector<LItem>> per(grid);
  size_t slot = 0;
  int nitems = 0;
  int zt = 0;
  long long T0 = 0;
  // At least a full wave of tiles (large h): whole-K tiles, tile i on CTA i mod grid.  The CTAs of
  // a wave then walk the same k-blocks in step and share their A / B blocks in L2 (a stream-K
  // split would start every CTA at another k and stream the operands from DRAM once per tile).
  const bool waves = (int)tiles.size() >= grid && grid == kLMaxCta;
  for (int ti = 0; waves && ti < (int)tiles.size(); ++ti) {
    LItem it{};
    it.gtile = (unsigned short)ti; it.ltile = (unsigned short)tiles[ti].ltile; it.job = (unsigned char)tiles[ti].job;
    it.npiece = 1; it.g0 = 0; it.g1 = (int)tiles[ti].w;
    per[ti % grid].push_back(it);
    ++nitems;
  }
  for (int ti = 0; !waves && ti < (int)tiles.size(); ++ti) {
    const T& t = tiles[ti];
    LItem it{};
    it.gtile = (unsigned short)ti; it.ltile = (unsigned short)t.ltile; it.job = (unsigned char)t.job;
    if (t.w == 0) {                                       // no work: one piece writes zeros
      it.npiece = 1; it.g0 = it.g1 = 0;
      per[zt++ % grid].push_back(it);
      ++nitems;
      continue;
    }
    const long long T1 = T0 + t.w;
    // CTA c owns [c W / grid, (c + 1) W / grid)
    auto owner = [&](long long g) { return (int)std::min<long long>(grid - 1, (g * grid) / W); };
    int c = owner(T0);
    while ((long long)(c + 1) * W / grid <= T0) ++c;
    std::vector<std::pair<int, std::pair<long long, long long>>> pcs;
    long long g = T0;
    while (g < T1) {
      const long long e = std::min(T1, (long long)(c + 1) * W / grid);
      if (e > g) pcs.push_back({c, {g, e}});
      g = e;
      ++c;
    }
    if (pcs.size() > 255) return false;
    it.npiece = (unsigned char)pcs.size();
    it.slot = (unsigned short)slot;
    if (pcs.size() > 1) slot += pcs.size();
    for (size_t p = 0; p < pcs.size(); ++p) {
      LItem q = it;
      q.piece = (unsigned char)p;
      q.g0 = (int)(pcs[p].second.first - T0);
      q.g1 = (int)(pcs[p].second.second - T0);
      per[pcs[p].first].push_back(q);
      ++nitems;
    }
    T0 = T1;
  }
  if (nitems > kLMaxItems || slot > l->slots || slot > 65535) return false;
  P.nitems = 0;
  for (int c = 0; c < grid; ++c) {
    P.cta_start[c] = (unsigned short)P.nitems;
    for (const LItem& it : per[c]) P.item[P.nitems++] = it;
  }
  P.cta_start[grid] = (unsigned short)P.nitems;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kLThreads, 1, 1);
  cfg.dynamicSmemBytes = kLSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_lazy, l->A_dz, l->B_hk, l->B_xp, D, P) == cudaSuccess;
}

}  // namespace cavs
