// skinny.cu — level kernel for SMALL tasks (M_t <= kSkinnyMax vertices), both precisions.
//
// A task of a few vertices is bound by streaming F's weights (2-8 MB) through the SMs, not by
// math: the tensor-core kernel puts 128 units per CTA, i.e. only h/128 CTAs each pulling
// 0.5-1 MB.  Here a CTA owns kUnits = 4 units of every gate, so the weights spread over h/4
// CTAs (~16 KB each, read once from L2), the task's operand rows are staged in shared memory
// and the K loop is split across lanes/warps with fp32 accumulation and a shuffle reduction.
// Numerics are those of the selected precision (bf16 operands incl. the bf16 child sum h~,
// fp32 accumulate), so results match the tensor-core path up to summation order.  The fused
// epilogue is the same cells.cuh code as every other level kernel.
#include "cells.cuh"
#include "kernels.h"

namespace cavs {

constexpr int kUnits = 4;          // units of each gate per CTA
constexpr int kKC = 256;           // K chunk staged in shared memory (static smem < 48 KB)
constexpr int kSkThreads = 256;    // 8 warps: warp w -> row (w % 4), K half (w / 4)

template <class OpT, int NACC, int E>
__global__ void __launch_bounds__(kSkThreads) k_skinny(Dev D, SegListI L, int row_lo, int row_hi, int units) {
  __shared__ float Bs[kSkinnyMax][kKC + 1];
  __shared__ float part[2][kUnits][kSkinnyMax];
  __shared__ float out[NACC][kUnits][kSkinnyMax];
  __shared__ VMeta s_meta[kSkinnyMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = blockIdx.x * kUnits;
  const int M = row_hi - row_lo;
  if (threadIdx.x < M) load_meta(D, row_lo + threadIdx.x, epi_needs_children<E>(), s_meta[threadIdx.x]);
  for (int i = threadIdx.x; i < NACC * kUnits * kSkinnyMax; i += kSkThreads) (&out[0][0][0])[i] = 0.f;
  const int row = warp & (kUnits - 1), khalf = warp >> 2;
  for (int si = 0; si < L.n; ++si) {
    const SegI s = L.s[si];
    const OpT* A = reinterpret_cast<const OpT*>(s.A);
    const bool write_hs = s.b_src == B_HSUM && blockIdx.x == 0 && D.Hs != nullptr;
    float acc[kSkinnyMax];
#pragma unroll
    for (int v = 0; v < kSkinnyMax; ++v) acc[v] = 0.f;
    const int j = u0 + row;
    for (int k0 = 0; k0 < s.klen; k0 += kKC) {
      const int kc = min(kKC, s.klen - k0);
      __syncthreads();
      for (int e = threadIdx.x; e < M * kc; e += kSkThreads) {
        const int v = e / kc, k = e % kc, p = row_lo + v;
        float b;
        if (s.b_src == B_HSUM) {                 // child sum h~ as the tensor-core path forms it
          const OpT* hk = reinterpret_cast<const OpT*>(D.Hk) + (size_t)p * D.N * D.h + k0 + k;
          float t = 0.f;
          for (int q = 0; q < D.N; ++q) t += from_op(hk[q * D.h]);
          const OpT r = to_op<OpT>(t);
          b = from_op(r);
          if (write_hs) reinterpret_cast<OpT*>(D.Hs)[(size_t)p * D.h + k0 + k] = r;
        } else {
          const OpT* base = reinterpret_cast<const OpT*>(s.b_src == B_HK ? D.Hk : s.b_src == B_XP ? D.Xp : D.dZ);
          b = from_op(base[(size_t)p * s.ldb + s.b_col + k0 + k]);
        }
        Bs[v][k] = b;
      }
      __syncthreads();
      if (j < units) {
        const OpT* a = A + (size_t)(s.a_row + j) * s.lda + k0;
        for (int k = khalf * 32 + lane; k < kc; k += 64) {
          const float w = from_op(a[k]);
#pragma unroll
          for (int v = 0; v < kSkinnyMax; ++v) acc[v] = fmaf(w, Bs[v][k], acc[v]);
        }
      }
    }
    // reduce over lanes, then over the two K halves
#pragma unroll
    for (int v = 0; v < kSkinnyMax; ++v) {
      float x = acc[v];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) part[khalf][row][v] = x;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kUnits * kSkinnyMax; i += kSkThreads) {
      const int r = i / kSkinnyMax, v = i % kSkinnyMax;
      out[s.acc][r][v] += part[0][r][v] + part[1][r][v];
    }
  }
  __syncthreads();
  // fused epilogue: thread -> (unit r, vertex v)
  for (int i = threadIdx.x; i < kUnits * M; i += kSkThreads) {
    const int r = i / M, v = i % M;
    const int j = u0 + r;
    const int p = row_lo + v;
    if (j >= units || !row_active<E>(D, p, s_meta[v].xrow)) continue;
    const UnitC uc = epi_uses_bias<E>() ? load_unit(D, j, epi_is_lstm<E>()) : UnitC{0.f, 0.f, 0.f, 0.f};
    float a[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) a[q] = out[q][r][v];
    typename EpiK<E>::In in;
    EpiK<E>::load(D, j, s_meta[v], in);
    EpiK<E>::template store<OpT>(D, j, s_meta[v], a, in, uc);
  }
}

template <class OpT, int NACC, int E>
static void sk(const Dev& D, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s) {
  k_skinny<OpT, NACC, E><<<cdiv(units, kUnits), kSkThreads, 0, s>>>(D, L, row_lo, row_hi, units);
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
    default: break;
  }
}

template void skinny_typeI<float>(const Dev&, int, const SegListI&, int, int, int, cudaStream_t);
template void skinny_typeI<__nv_bfloat16>(const Dev&, int, const SegListI&, int, int, int, cudaStream_t);

}  // namespace cavs
