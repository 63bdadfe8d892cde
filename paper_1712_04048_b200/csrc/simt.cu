// simt.cu — FP32 mode: FFMA (SIMT) level kernels with the fused cell epilogue, and the
// lazily batched weight-gradient GEMMs (§3.5 lazy batching).
//
// Type I  ("weights x task rows"): out[unit j, position p] = sum_seg A_seg[a_row + j, :] . B_seg[p, :]
//          over the positions of one task V_t, accumulators fed to the cell epilogue (cells.cuh).
// Type II ("lazy reduction over positions"): out[m, n] = sum_seg sum_p A_seg[p, a_col+m] * B_seg[p, b_col+n].
#include "cells.cuh"
#include "kernels.h"

namespace cavs {

constexpr int ST = 32;   // tile edge

template <class OpT>
__device__ __forceinline__ float load_b(const Dev& D, const SegI& s, int p, int k) {
  const OpT* base = reinterpret_cast<const OpT*>(s.b_src == B_HK ? D.Hk : s.b_src == B_XP ? D.Xp : D.dZ);
  return from_op(base[(size_t)p * s.ldb + s.b_col + k]);
}

template <class OpT, int NACC, int E>
__global__ void __launch_bounds__(256) k_simt_typeI(Dev D, SegListI L, int row_lo, int row_hi, int units) {
  __shared__ float As[ST][ST + 1];   // [k][unit]
  __shared__ float Bs[ST][ST + 1];   // [pos][k]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j0 = blockIdx.x * ST, p0 = row_lo + blockIdx.y * ST;
  // tile skipping: no row of this tile needs the epilogue
  {
    bool act = false;
    if (threadIdx.x < ST) { const int p = p0 + threadIdx.x; act = p < row_hi && row_active<E>(D, p, D.xrow_pos[p]); }
    if (!__syncthreads_or(act)) return;
  }
  float acc[NACC][4];
#pragma unroll
  for (int a = 0; a < NACC; ++a)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[a][r] = 0.f;

  for (int si = 0; si < L.n; ++si) {
    const SegI s = L.s[si];
    const OpT* A = reinterpret_cast<const OpT*>(s.A);
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k0 = 0; k0 < s.klen; k0 += ST) {
      for (int e = threadIdx.x; e < ST * ST; e += 256) {
        const int u = e >> 5, k = e & 31;
        const int j = j0 + u;
        As[k][u] = (j < units && k0 + k < s.klen) ? from_op(A[(size_t)(s.a_row + j) * s.lda + k0 + k]) : 0.f;
        const int p = p0 + u;
        float bv = 0.f;
        if (p < row_hi && k0 + k < s.klen) bv = load_b<OpT>(D, s, p, k0 + k);
        Bs[u][k] = bv;
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < ST; ++k) {
        const float a = As[k][tx];
#pragma unroll
        for (int r = 0; r < 4; ++r) t[r] = fmaf(a, Bs[ty + 8 * r][k], t[r]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < NACC; ++a)
      if (a == s.acc)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[a][r] += t[r];
  }
  const int j = j0 + tx;
  if (j >= units) return;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int p = p0 + ty + 8 * r;
    if (p >= row_hi) continue;
    VMeta m;
    load_meta(D, p, epi_needs_children<E>(), m);
    if (!row_active<E>(D, p, m.xrow)) continue;
    float v[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) v[a] = acc[a][r];
    epilogue1<E, OpT, NACC>(D, j, m, v);
  }
}

template <class OpT>
__global__ void __launch_bounds__(256) k_simt_typeII(Dev D, SegListII L, float* out, int M, int Ncols, int ldo,
                                                     int accum) {
  __shared__ float As[ST][ST + 1];   // [pos][m]
  __shared__ float Bs[ST][ST + 1];   // [pos][n]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int m0 = blockIdx.x * ST, n0 = blockIdx.y * ST;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int si = 0; si < L.n; ++si) {
    const SegII s = L.s[si];
    const OpT* A = reinterpret_cast<const OpT*>(s.A);
    const OpT* B = reinterpret_cast<const OpT*>(s.B);
    for (int q0 = s.k_lo; q0 < s.k_hi; q0 += ST) {
      if (s.skip_no_x) {
        const int t0 = q0 >> 6, t1 = min(q0 + ST - 1, s.k_hi - 1) >> 6;
        if (!D.tile_x[t0] && !D.tile_x[t1]) continue;        // uniform across the CTA
      }
      for (int e = threadIdx.x; e < ST * ST; e += 256) {
        const int r = e >> 5, c = e & 31;
        const int q = q0 + r;
        const bool ok = q < s.k_hi;
        As[r][c] = (ok && m0 + c < M) ? from_op(A[(size_t)q * s.lda + s.a_col + m0 + c]) : 0.f;
        Bs[r][c] = (ok && n0 + c < Ncols) ? from_op(B[(size_t)q * s.ldb + s.b_col + n0 + c]) : 0.f;
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < ST; ++k) {
        const float a = As[k][tx];
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] = fmaf(a, Bs[k][ty + 8 * r], acc[r]);
      }
      __syncthreads();
    }
  }
  const int m = m0 + tx;
  if (m >= M) return;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int n = n0 + ty + 8 * r;
    if (n < Ncols) out[(size_t)m * ldo + n] = accum ? out[(size_t)m * ldo + n] + acc[r] : acc[r];
  }
}

template <class OpT, int NACC, int E>
static void typeI(const Dev& D, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  dim3 grid(cdiv(units, ST), cdiv(row_hi - row_lo, ST));
  k_simt_typeI<OpT, NACC, E><<<grid, 256, 0, s>>>(D, L, row_lo, row_hi, units);
}

template <class OpT>
void simt_typeI(const Dev& D, int epi, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s) {
  switch (epi) {
    case EPI_LSTM_XPROJ: typeI<OpT, 4, EPI_LSTM_XPROJ>(D, L, row_lo, row_hi, units, s); break;
    case EPI_LSTM_FWD:
      if (D.N == 1) typeI<OpT, 4, EPI_LSTM_FWD>(D, L, row_lo, row_hi, units, s);
      else if (D.N == 2) typeI<OpT, 5, EPI_LSTM_FWD>(D, L, row_lo, row_hi, units, s);
      else typeI<OpT, 3 + kMaxN, EPI_LSTM_FWD>(D, L, row_lo, row_hi, units, s);
      break;
    case EPI_LSTM_BWD:
      if (D.N == 1) typeI<OpT, 2, EPI_LSTM_BWD>(D, L, row_lo, row_hi, units, s);
      else if (D.N == 2) typeI<OpT, 3, EPI_LSTM_BWD>(D, L, row_lo, row_hi, units, s);
      else typeI<OpT, 1 + kMaxN, EPI_LSTM_BWD>(D, L, row_lo, row_hi, units, s);
      break;
    case EPI_FC_XPROJ: typeI<OpT, 1, EPI_FC_XPROJ>(D, L, row_lo, row_hi, units, s); break;
    case EPI_FC_FWD: typeI<OpT, 1, EPI_FC_FWD>(D, L, row_lo, row_hi, units, s); break;
    case EPI_FC_BWD: typeI<OpT, 2, EPI_FC_BWD>(D, L, row_lo, row_hi, units, s); break;
    case EPI_LSTM_BWD_DAG:
      if (D.N == 1) typeI<OpT, 2, EPI_LSTM_BWD_DAG>(D, L, row_lo, row_hi, units, s);
      else if (D.N == 2) typeI<OpT, 3, EPI_LSTM_BWD_DAG>(D, L, row_lo, row_hi, units, s);
      else typeI<OpT, 1 + kMaxN, EPI_LSTM_BWD_DAG>(D, L, row_lo, row_hi, units, s);
      break;
    case EPI_FC_BWD_DAG: typeI<OpT, 2, EPI_FC_BWD_DAG>(D, L, row_lo, row_hi, units, s); break;
    default: typeI<OpT, 1, EPI_DX>(D, L, row_lo, row_hi, units, s); break;
  }
}

template <class OpT>
void simt_typeII(const Dev& D, const SegListII& L, float* out, int M, int Ncols, int ldo, cudaStream_t s, int accum) {
  dim3 grid(cdiv(M, ST), cdiv(Ncols, ST));
  k_simt_typeII<OpT><<<grid, 256, 0, s>>>(D, L, out, M, Ncols, ldo, accum);
}

SegListI fwd_segments(const Dev& D) {
  const int h = D.h, N = D.N;
  SegListI F{};
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    // U_g h~ = sum_k U_g h_k (linearity, reading Z11): one segment per (gate, child slot)
    F.n = 0;
    for (int g = 0; g < 3; ++g)
      for (int k = 0; k < N; ++k) F.s[F.n++] = SegI{D.Wa, h, g * h, B_HK, k * h, N * h, h, g};
    for (int k = 0; k < N; ++k) F.s[F.n++] = SegI{D.Wa, h, 3 * h, B_HK, k * h, N * h, h, 3 + k};
  } else {
    F.n = 1;
    F.s[0] = SegI{D.Wa, 2 * h, 0, B_HK, 0, 2 * h, 2 * h, 0};
  }
  return F;
}

SegListI bwd_segments(const Dev& D) {
  const int h = D.h, N = D.N;
  SegListI B{};
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    const int G = 3 + N;
    B.n = 1 + N;
    B.s[0] = SegI{D.Wc, 3 * h, 0, B_DZ, 0, G * h, 3 * h, 0};
    for (int k = 0; k < N; ++k) B.s[1 + k] = SegI{D.Wd, h, 0, B_DZ, (3 + k) * h, G * h, h, 1 + k};
  } else {
    B.n = 2;
    for (int k = 0; k < 2; ++k) B.s[k] = SegI{D.Wc, h, k * h, B_DZ, 0, h, h, k};
  }
  return B;
}

// ---- whole passes (FP32 mode; BF16 operands when CAVS_BF16_SIMT=1 for A/B checks) ----
template <class OpT>
void simt_forward(Dev& D, const std::vector<int>& lp, cudaStream_t s, Prof& P, XStream* xs) {
  const int skmax = skinny_max(D);
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  SegListI L{}, F{};
  if (lstm) {
    L.n = 4;
    for (int g = 0; g < 4; ++g) L.s[g] = SegI{D.Wb, d, g * h, B_XP, 0, d, d, g};
  } else {
    L.n = 1;
    L.s[0] = SegI{D.Wb, d, 0, B_XP, 0, d, d, 0};
  }
  const int xepi = lstm ? EPI_LSTM_XPROJ : EPI_FC_XPROJ, fepi = lstm ? EPI_LSTM_FWD : EPI_FC_FWD;
  // eager x-projection; streaming ablation: the rows above level 0 on a second
  // stream, task t waiting only for its own rows
  const bool streamed = D.stream_x && xs && xs->s;
  if (streamed) {
    while ((int)xs->ev.size() < T) { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); xs->ev.push_back(e); }
    cudaEventRecord(xs->start, s);
    cudaStreamWaitEvent(xs->s, xs->start, 0);
    for (int t = 1; t < T; ++t) {
      simt_typeI<OpT>(D, xepi, L, lp[t], lp[t + 1], h, xs->s);
      cudaEventRecord(xs->ev[t], xs->s);
    }
    simt_typeI<OpT>(D, xepi, L, 0, T > 1 ? lp[1] : D.V, h, s);
    P.count(T);
  } else {
    simt_typeI<OpT>(D, xepi, L, 0, D.V, h, s); P.count(1);
  }
  P.mark(CAVS_PH_FWD_LEVELS, s);
  F = fwd_segments(D);
  for (int t = 1; t < T; ++t) {
    if (D.dag) { launch_dag_gather(D, lp[t], lp[t + 1], s); P.count(1); }
    if (streamed) cudaStreamWaitEvent(s, xs->ev[t], 0);
    if (lp[t + 1] - lp[t] <= skmax) skinny_typeI<OpT>(D, fepi, F, lp[t], lp[t + 1], h, s);
    else simt_typeI<OpT>(D, fepi, F, lp[t], lp[t + 1], h, s);
    P.count(1);
    if (D.unfused) { launch_unfused(D, fepi, lp[t], lp[t + 1], s); P.count(1); }
  }
}

template <class OpT>
void simt_backward(Dev& D, const std::vector<int>& lp, cudaStream_t s, Prof& P) {
  const int skmax = skinny_max(D);
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int G = lstm ? 3 + N : 1;
  SegListI B{};
  int epi;
  if (lstm) {
    B.n = 1 + N;
    B.s[0] = SegI{D.Wc, 3 * h, 0, B_DZ, 0, G * h, 3 * h, 0};
    for (int k = 0; k < N; ++k) B.s[1 + k] = SegI{D.Wd, h, 0, B_DZ, (3 + k) * h, G * h, h, 1 + k};
    epi = EPI_LSTM_BWD;
  } else {
    B.n = 2;
    for (int k = 0; k < 2; ++k) B.s[k] = SegI{D.Wc, h, k * h, B_DZ, 0, h, h, k};
    epi = EPI_FC_BWD;
  }
  if (D.dag) {                      // DAG batch: pull-reduce + dF per task, then the edge gradients
    epi = lstm ? EPI_LSTM_BWD_DAG : EPI_FC_BWD_DAG;
    for (int t = T - 1; t >= 0; --t) {
      launch_dag_df(D, lp[t], lp[t + 1], s);
      P.count(1);
      if (t == 0) break;
      if (lp[t + 1] - lp[t] <= skmax) skinny_typeI<OpT>(D, epi, B, lp[t], lp[t + 1], h, s);
      else simt_typeI<OpT>(D, epi, B, lp[t], lp[t + 1], h, s);
      P.count(1);
      if (D.unfused) { launch_unfused(D, epi, lp[t], lp[t + 1], s); P.count(1); }
    }
  } else {
  for (int t = T - 1; t >= 1; --t) {
    if (lp[t + 1] - lp[t] <= skmax) skinny_typeI<OpT>(D, epi, B, lp[t], lp[t + 1], h, s);
    else simt_typeI<OpT>(D, epi, B, lp[t], lp[t + 1], h, s);
    P.count(1);
    if (D.unfused) { launch_unfused(D, epi, lp[t], lp[t + 1], s); P.count(1); }
  }
  }
  P.mark(CAVS_PH_LAZY, s);
  // lazy batching of the parameter gradients over ALL vertices; one partial each
  const LazyLayout Z = lazy_layout(D);
  const int lp1 = D.lp1, V = D.V;
  if (D.lazy_off) {
    // ablation "lazy batching off": one set of weight-gradient GEMMs per task over its own
    // rows, accumulated in stream order
    for (int t = 0; t < T; ++t) {
      const int lo = lp[t], hi = lp[t + 1], acc = t > 0 ? 1 : 0, accU = t > 1 ? 1 : 0;
      if (lstm) {
        if (t >= 1) {
          SegListII A{}; A.n = N;
          for (int k = 0; k < N; ++k) A.s[k] = SegII{D.dZ, G * h, 0, D.Hk, N * h, k * h, lo, hi, 0};
          simt_typeII<OpT>(D, A, D.lazy + Z.u4, 3 * h, h, h, s, accU);
          SegListII Bf{}; Bf.n = N;
          for (int k = 0; k < N; ++k) Bf.s[k] = SegII{D.dZ, G * h, (3 + k) * h, D.Hk, N * h, k * h, lo, hi, 0};
          simt_typeII<OpT>(D, Bf, D.lazy + Z.uf, h, h, h, s, accU);
          P.count(2);
        }
        SegListII Cw{}; Cw.n = 1;
        Cw.s[0] = SegII{D.dZ, G * h, 0, D.Xp, d, 0, lo, hi, 1};
        simt_typeII<OpT>(D, Cw, D.lazy + Z.w, G * h, d, d, s, acc);
      } else {
        if (t >= 1) {
          SegListII A{}; A.n = 1;
          A.s[0] = SegII{D.dZ, h, 0, D.Hk, 2 * h, 0, lo, hi, 0};
          simt_typeII<OpT>(D, A, D.lazy + Z.u4, h, 2 * h, 2 * h, s, accU);
          P.count(1);
        }
        SegListII Cw{}; Cw.n = 1;
        Cw.s[0] = SegII{D.dZ, h, 0, D.Xp, d, 0, lo, hi, 1};
        simt_typeII<OpT>(D, Cw, D.lazy + Z.w, h, d, d, s, acc);
      }
      P.count(1);
    }
    if (T <= 1) {
      cudaMemsetAsync(D.lazy + Z.u4, 0, sizeof(float) * Z.su4, s);
      if (lstm) cudaMemsetAsync(D.lazy + Z.uf, 0, sizeof(float) * Z.suf, s);
    }
  } else if (lstm) {
    SegListII A{}; A.n = N;                      // dU_iou = sum_k dZ_iou^T H_k
    for (int k = 0; k < N; ++k) A.s[k] = SegII{D.dZ, G * h, 0, D.Hk, N * h, k * h, lp1, V, 0};
    simt_typeII<OpT>(D, A, D.lazy + Z.u4, 3 * h, h, h, s, 0);
    SegListII Bf{}; Bf.n = N;
    for (int k = 0; k < N; ++k) Bf.s[k] = SegII{D.dZ, G * h, (3 + k) * h, D.Hk, N * h, k * h, lp1, V, 0};
    simt_typeII<OpT>(D, Bf, D.lazy + Z.uf, h, h, h, s, 0);
    SegListII Cw{}; Cw.n = 1;
    Cw.s[0] = SegII{D.dZ, G * h, 0, D.Xp, d, 0, 0, V, 1};
    simt_typeII<OpT>(D, Cw, D.lazy + Z.w, G * h, d, d, s, 0);
    P.count(3);
  } else {
    SegListII A{}; A.n = 1;
    A.s[0] = SegII{D.dZ, h, 0, D.Hk, 2 * h, 0, lp1, V, 0};
    simt_typeII<OpT>(D, A, D.lazy + Z.u4, h, 2 * h, 2 * h, s, 0);
    SegListII Cw{}; Cw.n = 1;
    Cw.s[0] = SegII{D.dZ, h, 0, D.Xp, d, 0, 0, V, 1};
    simt_typeII<OpT>(D, Cw, D.lazy + Z.w, h, d, d, s, 0);
    P.count(2);
  }
  P.mark(CAVS_PH_DX, s);
  if (D.dx) {
    SegListI X{}; X.n = 1;
    X.s[0] = SegI{D.We, G * h, 0, B_DZ, 0, G * h, G * h, 0};
    simt_typeI<OpT>(D, EPI_DX, X, 0, V, d, s); P.count(1);
  }
}

template void simt_forward<float>(Dev&, const std::vector<int>&, cudaStream_t, Prof&, XStream*);
template void simt_forward<__nv_bfloat16>(Dev&, const std::vector<int>&, cudaStream_t, Prof&, XStream*);
template void simt_backward<float>(Dev&, const std::vector<int>&, cudaStream_t, Prof&);
template void simt_backward<__nv_bfloat16>(Dev&, const std::vector<int>&, cudaStream_t, Prof&);

template void simt_typeI<float>(const Dev&, int, const SegListI&, int, int, int, cudaStream_t);
template void simt_typeI<__nv_bfloat16>(const Dev&, int, const SegListI&, int, int, int, cudaStream_t);
template void simt_typeII<float>(const Dev&, const SegListII&, float*, int, int, int, cudaStream_t, int);
template void simt_typeII<__nv_bfloat16>(const Dev&, const SegListII&, float*, int, int, int, cudaStream_t, int);

}  // namespace cavs
