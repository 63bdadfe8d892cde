// cells.cuh — the vertex function F and its derivative dF as per-(unit j, position p)
// epilogues, shared by the FP32 (FFMA) and BF16 (tcgen05) level kernels.
//
// Tree-LSTM, N-ary child-sum (Fig. 5):
//   h~ = sum_k h_k; i = s(W_i x + U_i h~ + b_i); f_k = s(W_f x + U_f h_k + b_f);
//   o = s(W_o x + U_o h~ + b_o); u = tanh(W_u x + U_u h~ + b_u);
//   c = i*u + sum_k f_k*c_k; h = o*tanh(c); scatter [c,h]; push h.
// Tree-FC (reading Z7): h = tanh(W_c [h_l; h_r] + W_x x + b).
// Backward: hand-derived dF (checked by FD in tests/test_oracle_pins.py);
// gradients flowing to children are written by the unique parent (forests), i.e. the
// "added" of P:L447 is a plain store because every child has exactly one adder.
//
// Internal gate order of every per-vertex row: (i, o, u, f_1..f_N); weights/bias are
// repacked to it by k_prep (see ops.cu).
#pragma once
#include "kernels.h"

namespace cavs {

template <class OpT> __device__ __forceinline__ OpT* op(void* p) { return reinterpret_cast<OpT*>(p); }

// ---- Tree-LSTM --------------------------------------------------------------
// Finish F at (j, p) given gate pre-activations (bias already added).
template <class OpT>
__device__ __forceinline__ void lstm_finish(const Dev& D, int j, int p, float zi, float zo, float zu,
                                            const float* zf) {
  const int h = D.h, N = D.N, G = 3 + N;
  const float i = sigm(zi), o = sigm(zo), u = tanhf(zu);
  float c = i * u;
  const int deg = D.deg[p];
  float* g = D.gates + (size_t)p * G * h;
  const float* ck = D.Ck + (size_t)p * N * h;
  for (int k = 0; k < N; ++k) {
    const float f = sigm(zf[k]);
    g[(3 + k) * h + j] = f;
    if (k < deg) c += f * ck[k * h + j];          // missing children: c_k = 0 (Z1)
  }
  const float hv = o * tanhf(c);
  g[j] = i; g[h + j] = o; g[2 * h + j] = u;
  D.cst[(size_t)p * h + j] = c;
  D.h_out[(size_t)D.order[p] * h + j] = hv;      // push(h)
  const int par = D.parent_pos[p];
  if (par >= 0) {                                // scatter([c,h]) into the parent's gather slot
    const size_t at = (size_t)par * N * h + (size_t)D.slot[p] * h + j;
    op<OpT>(D.Hk)[at] = to_op<OpT>(hv);
    D.Ck[at] = c;
  }
}

// Level kernel epilogue, t >= 1: acc = (U_i h~, U_o h~, U_u h~, U_f h_1..U_f h_N).
template <class OpT>
__device__ __forceinline__ void epi_lstm_fwd(const Dev& D, int j, int p, const float* acc) {
  const int h = D.h;
  float xi = 0.f, xo = 0.f, xu = 0.f, xf = 0.f;
  if (D.xrow_pos[p] >= 0) {                      // eager pull projection
    const float* xw = D.XW + (size_t)p * 4 * h;
    xi = xw[j]; xo = xw[h + j]; xu = xw[2 * h + j]; xf = xw[3 * h + j];
  }
  const float* b = D.bias;
  float zf[8];
  for (int k = 0; k < D.N; ++k) zf[k] = acc[3 + k] + xf + b[3 * h + j];
  lstm_finish<OpT>(D, j, p, acc[0] + xi + b[j], acc[1] + xo + b[h + j], acc[2] + xu + b[2 * h + j], zf);
}

// Eager pull projection epilogue: acc = (W_i x, W_o x, W_u x, W_f x).  Level-0 vertices
// (no children, so no recurrent term) are finished here; x-vertices above level 0
// keep their projection for their own level.
template <class OpT>
__device__ __forceinline__ void epi_lstm_xproj(const Dev& D, int j, int p, const float* acc) {
  const int h = D.h;
  if (p < D.lp1) {
    const float* b = D.bias;
    float zf[8];
    for (int k = 0; k < D.N; ++k) zf[k] = acc[3] + b[3 * h + j];
    lstm_finish<OpT>(D, j, p, acc[0] + b[j], acc[1] + b[h + j], acc[2] + b[2 * h + j], zf);
  } else if (D.xrow_pos[p] >= 0) {
    float* xw = D.XW + (size_t)p * 4 * h;
    xw[j] = acc[0]; xw[h + j] = acc[1]; xw[2 * h + j] = acc[2]; xw[3 * h + j] = acc[3];
  }
}

// dF at position c, unit j, given dL/dh and dL/dc arriving from the parent (+ push's adjoint).
template <class OpT>
__device__ __forceinline__ void lstm_elem_bwd(const Dev& D, int j, int c, float dh, float dc) {
  const int h = D.h, N = D.N, G = 3 + N;
  const float* g = D.gates + (size_t)c * G * h;
  const float i = g[j], o = g[h + j], u = g[2 * h + j];
  const float tc = tanhf(D.cst[(size_t)c * h + j]);
  const float dzo = dh * tc * o * (1.f - o);
  const float dcb = dc + dh * o * (1.f - tc * tc);
  const float dzi = dcb * u * i * (1.f - i);
  const float dzu = dcb * i * (1.f - u * u);
  OpT* dz = op<OpT>(D.dZ) + (size_t)c * G * h;
  dz[j] = to_op<OpT>(dzi); dz[h + j] = to_op<OpT>(dzo); dz[2 * h + j] = to_op<OpT>(dzu);
  const int deg = D.deg[c];
  const float* ck = D.Ck + (size_t)c * N * h;
  for (int k = 0; k < N; ++k) {
    float v = 0.f;
    if (k < deg) { const float f = g[(3 + k) * h + j]; v = dcb * ck[k * h + j] * f * (1.f - f); }
    dz[(3 + k) * h + j] = to_op<OpT>(v);
  }
  D.dcb[(size_t)c * h + j] = dcb;
}

// Backward level epilogue at parent p: acc[0] = U_iou^T dz_iou (= dL/dh~), acc[1+k] = U_f^T dz_fk.
// Gather's adjoint: child k receives dh~ + U_f^T dz_fk and dc-bar * f_k.
template <class OpT>
__device__ __forceinline__ void epi_lstm_bwd(const Dev& D, int j, int p, const float* acc) {
  const int h = D.h, N = D.N;
  const int deg = D.deg[p];
  const float dcbp = D.dcb[(size_t)p * h + j];
  const float* g = D.gates + (size_t)p * (3 + N) * h;
  for (int k = 0; k < deg; ++k) {
    const int c = D.child_pos[(size_t)p * N + k];
    const float dh = acc[0] + acc[1 + k] + D.dh_out[(size_t)D.order[c] * h + j];
    lstm_elem_bwd<OpT>(D, j, c, dh, dcbp * g[(3 + k) * h + j]);
  }
}

// ---- Tree-FC ------------------------------------------------------------------
template <class OpT>
__device__ __forceinline__ void fc_finish(const Dev& D, int j, int p, float z) {
  const int h = D.h;
  const float hv = tanhf(z);
  D.gates[(size_t)p * h + j] = hv;
  D.h_out[(size_t)D.order[p] * h + j] = hv;
  const int par = D.parent_pos[p];
  if (par >= 0) op<OpT>(D.Hk)[(size_t)par * 2 * h + (size_t)D.slot[p] * h + j] = to_op<OpT>(hv);
}

template <class OpT>
__device__ __forceinline__ void epi_fc_fwd(const Dev& D, int j, int p, const float* acc) {
  const float xw = D.xrow_pos[p] >= 0 ? D.XW[(size_t)p * D.h + j] : 0.f;
  fc_finish<OpT>(D, j, p, acc[0] + xw + D.bias[j]);
}

template <class OpT>
__device__ __forceinline__ void epi_fc_xproj(const Dev& D, int j, int p, const float* acc) {
  if (p < D.lp1) fc_finish<OpT>(D, j, p, acc[0] + D.bias[j]);
  else if (D.xrow_pos[p] >= 0) D.XW[(size_t)p * D.h + j] = acc[0];
}

template <class OpT>
__device__ __forceinline__ void fc_elem_bwd(const Dev& D, int j, int c, float dh) {
  const float hv = D.gates[(size_t)c * D.h + j];
  op<OpT>(D.dZ)[(size_t)c * D.h + j] = to_op<OpT>(dh * (1.f - hv * hv));
}

// acc[k] = W_{l|r}^T dz  (k = 0: left, 1: right)
template <class OpT>
__device__ __forceinline__ void epi_fc_bwd(const Dev& D, int j, int p, const float* acc) {
  const int deg = D.deg[p];
  for (int k = 0; k < deg; ++k) {
    const int c = D.child_pos[(size_t)p * 2 + k];
    fc_elem_bwd<OpT>(D, j, c, acc[k] + D.dh_out[(size_t)D.order[c] * D.h + j]);
  }
}

// ---- pull's adjoint: dx ------------------------------------------------------------
__device__ __forceinline__ void epi_dx(const Dev& D, int j, int p, const float* acc) {
  const int r = D.xrow_pos[p];
  if (r >= 0) D.dx[(size_t)r * D.d + j] = acc[0];
}

template <int E, class OpT>
__device__ __forceinline__ void epilogue(const Dev& D, int j, int p, const float* acc) {
  if constexpr (E == EPI_LSTM_FWD) epi_lstm_fwd<OpT>(D, j, p, acc);
  else if constexpr (E == EPI_LSTM_XPROJ) epi_lstm_xproj<OpT>(D, j, p, acc);
  else if constexpr (E == EPI_LSTM_BWD) epi_lstm_bwd<OpT>(D, j, p, acc);
  else if constexpr (E == EPI_FC_FWD) epi_fc_fwd<OpT>(D, j, p, acc);
  else if constexpr (E == EPI_FC_XPROJ) epi_fc_xproj<OpT>(D, j, p, acc);
  else if constexpr (E == EPI_FC_BWD) epi_fc_bwd<OpT>(D, j, p, acc);
  else epi_dx(D, j, p, acc);
}

// Does position p need this epilogue at all? (tile skipping for the x-kernels)
template <int E>
__device__ __forceinline__ bool row_active(const Dev& D, int p) {
  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ) return p < D.lp1 || D.xrow_pos[p] >= 0;
  else if constexpr (E == EPI_DX) return D.xrow_pos[p] >= 0;
  else return true;
}

}  // namespace cavs
