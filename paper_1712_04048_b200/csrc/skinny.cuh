// skinny.cuh — level kernel for SMALL tasks (M_t <= kSkinnyMax vertices), both precisions.
//
// A task of a few vertices is bound by streaming F's weights (2-8 MB) through the SMs, not by
// math: the tensor-core kernel puts 128 units per CTA, i.e. only h/128 CTAs each pulling
// 0.5-1 MB.  Here a CTA owns kUnits = 4 units of every gate, so the weights spread over h/4
// CTAs (~16 KB each, read once from L2).  Each CTA stages the task's operand rows once in
// shared memory (16-byte vector loads; the child sum h~ is formed there, rounded like the
// tensor-core path), every warp loads its whole weight rows up front (one latency), and
// the K dot products run with fp32 accumulation and a shuffle reduction.  The fused
// epilogue is the same cells.cuh code as every other level kernel.
#pragma once
// (implementation shared by skinny_f32.cu / skinny_bf16.cu: one instantiation per translation unit,
// so the two heavily unrolled kernel sets compile in parallel)
#include "cells.cuh"
#include "kernels.h"

namespace cavs {

constexpr int kUnits = 4;          // units of each gate per CTA
constexpr int kSkThreads = 256;    // 8 warps

template <class OpT> struct Vec;   // 16-byte vector of operands
template <> struct Vec<float> { static constexpr int n = 4; };
template <> struct Vec<__nv_bfloat16> { static constexpr int n = 8; };

template <class OpT>
__device__ __forceinline__ void unpack16(const uint4& u, float* f) {
  if constexpr (sizeof(OpT) == 4) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y); f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  } else {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) { const float2 t = __bfloat1622float2(b[i]); f[2 * i] = t.x; f[2 * i + 1] = t.y; }
  }
}

// Staged operand layout (per vertex row, in OpT): the B source columns [0, W).
template <class OpT, int NACC, int E, int MV>
__global__ void __launch_bounds__(kSkThreads) k_skinny(Dev D, SegListI L, int row_lo, int row_hi, int units,
                                                      int bsrc, int W, int ldb) {
  constexpr int VE = Vec<OpT>::n;
  extern __shared__ __align__(16) uint8_t sk_smem[];
  OpT* Bs = reinterpret_cast<OpT*>(sk_smem);                    // [MV][W]
  float* out = reinterpret_cast<float*>(sk_smem + (size_t)MV * W * sizeof(OpT));   // [NACC][kUnits][MV]
  __shared__ VMeta s_meta[MV];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = blockIdx.x * kUnits;
  const int M = row_hi - row_lo;
  unsigned long long t_0 = 0, t_1 = 0, t_2 = 0;
  if (D.trace && threadIdx.x == 0) t_0 = gtime();
  if (threadIdx.x < M) load_meta(D, row_lo + threadIdx.x, epi_needs_children<E>(), s_meta[threadIdx.x]);
  asm volatile("griddepcontrol.wait;" ::: "memory");          // PDL: previous task complete + visible
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- stage the task's operand rows: all 16-byte copies in flight at once (cp.async) ----
  {
    const OpT* src = reinterpret_cast<const OpT*>(bsrc == B_HK ? D.Hk : bsrc == B_XP ? D.Xp : D.dZ);
    const int nv = W / VE;
    for (int e = threadIdx.x; e < MV * nv; e += kSkThreads) {
      const int v = e / nv, c = e % nv;
      OpT* dst = Bs + (size_t)v * W + c * VE;
      if (v < M) {
        const OpT* g = src + (size_t)(row_lo + v) * ldb + c * VE;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(g) : "memory");
      } else {
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  if (D.trace && threadIdx.x == 0) t_1 = gtime();
  // ---- dot products: row = (accumulator, unit); one warp sums all segments of its row ----
  for (int rr = warp; rr < NACC * kUnits; rr += kSkThreads / 32) {
    const int acc_id = rr / kUnits, r = rr % kUnits, j = u0 + r;
    if (j >= units) continue;                                   // warp-uniform
    float acc[MV];
#pragma unroll
    for (int v = 0; v < MV; ++v) acc[v] = 0.f;
    for (int si = 0; si < L.n; ++si) {
      const SegI s = L.s[si];
      if (s.acc != acc_id) continue;
      const OpT* a = reinterpret_cast<const OpT*>(s.A) + (size_t)(s.a_row + j) * s.lda;
      constexpr int KMAX = 12;                                  // vectors per lane kept in flight
      for (int kb = 0; kb < s.klen; kb += 32 * VE * KMAX) {
        uint4 av[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          const int k = kb + (i * 32 + lane) * VE;
          av[i] = k < s.klen ? *reinterpret_cast<const uint4*>(a + k) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          const int k = kb + (i * 32 + lane) * VE;
          if (k >= s.klen) break;
          float w[VE];
          unpack16<OpT>(av[i], w);
#pragma unroll
          for (int v = 0; v < MV; ++v) {
            float b[VE];
            unpack16<OpT>(*reinterpret_cast<const uint4*>(Bs + (size_t)v * W + s.b_col + k), b);
#pragma unroll
            for (int e = 0; e < VE; ++e) acc[v] = fmaf(w[e], b[e], acc[v]);
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < MV; ++v) {
      float x = acc[v];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) out[(acc_id * kUnits + r) * MV + v] = x;
    }
  }
  __syncthreads();
  if (D.trace && threadIdx.x == 0) t_2 = gtime();
  // ---- fused epilogue: thread -> (unit r, vertex v) ----
  for (int i = threadIdx.x; i < kUnits * M; i += kSkThreads) {
    const int r = i / M, v = i % M;
    const int j = u0 + r;
    const int p = row_lo + v;
    if (j >= units || !row_active<E>(D, p, s_meta[v].xrow)) continue;
    float av[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) av[q] = out[(q * kUnits + r) * MV + v];
    epilogue1<E, OpT, NACC>(D, j, s_meta[v], av);
  }
  if (D.trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long at = 8 + 8 * atomicAdd(D.trace, 1ull);
      if (at + 8 < (4u << 20) / 8) {
        D.trace[at] = 200 + E; D.trace[at + 1] = blockIdx.x; D.trace[at + 2] = row_lo;
        D.trace[at + 3] = t_0; D.trace[at + 4] = t_1; D.trace[at + 5] = t_2; D.trace[at + 6] = gtime();
        D.trace[at + 7] = row_hi;
      }
    }
  }
}

template <class OpT, int NACC, int E, int MV>
static void sk_mv(const Dev& D, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s) {
  // staged source: the union of the segments' B columns (all segments of a level kernel read one arena)
  int bsrc = B_DZ, W = 0, ldb = 0;
  for (int i = 0; i < L.n; ++i) {
    const SegI& g = L.s[i];
    bsrc = g.b_src; ldb = g.ldb; W = std::max(W, g.b_col + g.klen);
  }
  const size_t smem = (size_t)MV * W * sizeof(OpT) + (size_t)NACC * kUnits * MV * sizeof(float);
  static size_t attr[kMaxDev] = {};
  const int dv = cur_device();
  if (smem > 48 * 1024 && smem > attr[dv]) {
    cudaFuncSetAttribute(k_skinny<OpT, NACC, E, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[dv] = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cdiv(units, kUnits), 1, 1);
  cfg.blockDim = dim3(kSkThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL: overlap with the previous task
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_skinny<OpT, NACC, E, MV>, D, L, row_lo, row_hi, units, bsrc, W, ldb);
}

template <class OpT, int NACC, int E>
static void sk(const Dev& D, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s) {
  const int M = row_hi - row_lo;
  if (M <= 4) sk_mv<OpT, NACC, E, 4>(D, L, row_lo, row_hi, units, s);
  else if (M <= 8) sk_mv<OpT, NACC, E, 8>(D, L, row_lo, row_hi, units, s);
  else if (M <= 16) sk_mv<OpT, NACC, E, 16>(D, L, row_lo, row_hi, units, s);
  else sk_mv<OpT, NACC, E, 32>(D, L, row_lo, row_hi, units, s);
}

template <class OpT>
void skinny_typeI(const Dev& D, int epi, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  switch (epi) {
    case EPI_LSTM_FWD:
      if (D.N == 1) sk<OpT, 4, EPI_LSTM_FWD>(D, L, row_lo, row_hi, units, s);
      else if (D.N == 2) sk<OpT, 5, EPI_LSTM_FWD>(D, L, row_lo, row_hi, units, s);
      else sk<OpT, 3 + kMaxN, EPI_LSTM_FWD>(D, L, row_lo, row_hi, units, s);
      break;
    case EPI_LSTM_BWD:
      if (D.N == 1) sk<OpT, 2, EPI_LSTM_BWD>(D, L, row_lo, row_hi, units, s);
      else if (D.N == 2) sk<OpT, 3, EPI_LSTM_BWD>(D, L, row_lo, row_hi, units, s);
      else sk<OpT, 1 + kMaxN, EPI_LSTM_BWD>(D, L, row_lo, row_hi, units, s);
      break;
    case EPI_FC_FWD: sk<OpT, 1, EPI_FC_FWD>(D, L, row_lo, row_hi, units, s); break;
    case EPI_FC_BWD: sk<OpT, 2, EPI_FC_BWD>(D, L, row_lo, row_hi, units, s); break;
    case EPI_LSTM_BWD_DAG:
      if (D.N == 1) sk<OpT, 2, EPI_LSTM_BWD_DAG>(D, L, row_lo, row_hi, units, s);
      else if (D.N == 2) sk<OpT, 3, EPI_LSTM_BWD_DAG>(D, L, row_lo, row_hi, units, s);
      else sk<OpT, 1 + kMaxN, EPI_LSTM_BWD_DAG>(D, L, row_lo, row_hi, units, s);
      break;
    case EPI_FC_BWD_DAG: sk<OpT, 2, EPI_FC_BWD_DAG>(D, L, row_lo, row_hi, units, s); break;
    default: break;
  }
}


}  // namespace cavs
