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
// Every epilogue is split into load() (all global reads of one vertex, into registers)
// and store() (math + all writes), so a kernel can issue the loads of several vertices
// before the first store: the reads never alias the writes of the same launch (a task's
// own rows vs. its parents' / children's rows), and batching them turns a latency chain
// into memory-level parallelism.  Per-vertex metadata (VMeta) comes from shared memory
// in the tensor-core kernels.
//
// Internal gate order of every per-vertex row: (i, o, u, f_1..f_N); weights/bias are
// repacked to it by k_prep (see ops.cu).
#pragma once
#include "kernels.h"

namespace cavs {

template <class OpT> __device__ __forceinline__ OpT* op(void* p) { return reinterpret_cast<OpT*>(p); }

// Activations.  FP32 mode: accurate expf/tanhf (parity 1e-5).  BF16 mode: the MUFU tanh
// (tanh.approx.f32, rel. err <= 2^-10.99), sigmoid(z) = 0.5 tanh(z/2) + 0.5 — an order of
// magnitude below the bf16 operand rounding the mode already accepts (reading Z11).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <class OpT> __device__ __forceinline__ float act_sig(float z) {
  if constexpr (sizeof(OpT) == 2) return fmaf(0.5f, tanh_fast(0.5f * z), 0.5f);
  else return sigm(z);
}
template <class OpT> __device__ __forceinline__ float act_tanh(float z) {
  if constexpr (sizeof(OpT) == 2) return tanh_fast(z);
  else return tanhf(z);
}

struct VMeta {
  int p, vid, par, slot, deg, xrow;
  int ch[kMaxN], ch_vid[kMaxN], ch_deg[kMaxN];
};

__device__ __forceinline__ void load_meta(const Dev& D, int p, bool children, VMeta& m) {
  m.p = p;
  m.vid = D.order[p];
  m.par = D.parent_pos[p];
  m.slot = D.slot[p];
  m.deg = D.deg[p];
  m.xrow = D.xrow_pos[p];
#pragma unroll
  for (int k = 0; k < kMaxN; ++k) {
    const int c = (children && k < D.N) ? D.child_pos[(size_t)p * D.N + k] : -1;
    m.ch[k] = c;
    m.ch_vid[k] = c >= 0 ? D.order[c] : 0;
    m.ch_deg[k] = c >= 0 ? D.deg[c] : 0;
  }
}

// Per-unit constants (bias in the internal gate order), loaded once per thread.
struct UnitC { float b0, b1, b2, b3; };
__device__ __forceinline__ UnitC load_unit(const Dev& D, int j, bool lstm) {
  UnitC u;
  if (lstm) { u.b0 = D.bias[j]; u.b1 = D.bias[D.h + j]; u.b2 = D.bias[2 * D.h + j]; u.b3 = D.bias[3 * D.h + j]; }
  else { u.b0 = D.bias[j]; u.b1 = u.b2 = u.b3 = 0.f; }
  return u;
}

// ---- Tree-LSTM helpers -----------------------------------------------------------
template <class OpT>
__device__ __forceinline__ void lstm_finish(const Dev& D, int j, const VMeta& m, float zi, float zo, float zu,
                                            const float* zf, const float* ck) {
  const int h = D.h, N = D.N, G = 3 + N;
  const float i = act_sig<OpT>(zi), o = act_sig<OpT>(zo), u = act_tanh<OpT>(zu);
  float c = i * u;
  float* g = D.gates + (size_t)m.p * G * h;
#pragma unroll
  for (int k = 0; k < kMaxN; ++k) {
    if (k >= N) break;
    const float f = act_sig<OpT>(zf[k]);
    g[(3 + k) * h + j] = f;
    if (k < m.deg) c += f * ck[k];               // missing children: c_k = 0 (Z1)
  }
  const float hv = o * act_tanh<OpT>(c);
  g[j] = i; g[h + j] = o; g[2 * h + j] = u;
  D.cst[(size_t)m.p * h + j] = c;
  D.h_out[(size_t)m.vid * h + j] = hv;           // push(h)
  if (m.par >= 0) {                              // scatter([c,h]) into the parent's gather slot
    const size_t at = (size_t)m.par * N * h + (size_t)m.slot * h + j;
    op<OpT>(D.Hk)[at] = to_op<OpT>(hv);
    D.Ck[at] = c;
  }
}

// dF at child c (unit j): inputs already loaded.
struct LstmChildIn { float dho, i, o, u, cc; float f[kMaxN]; float ck[kMaxN]; };

__device__ __forceinline__ void lstm_child_load(const Dev& D, int j, int c, int c_vid, int c_deg, LstmChildIn& in) {
  const int h = D.h, N = D.N, G = 3 + N;
  const float* g = D.gates + (size_t)c * G * h;
  in.dho = D.dh_out[(size_t)c_vid * h + j];
  in.i = g[j]; in.o = g[h + j]; in.u = g[2 * h + j];
  in.cc = D.cst[(size_t)c * h + j];
  const float* ck = D.Ck + (size_t)c * N * h;
#pragma unroll
  for (int k = 0; k < kMaxN; ++k) {
    const bool have = k < c_deg;
    in.f[k] = have ? g[(3 + k) * h + j] : 0.f;
    in.ck[k] = have ? ck[k * h + j] : 0.f;
  }
}

template <class OpT>
__device__ __forceinline__ void lstm_child_store(const Dev& D, int j, int c, int c_deg, float dh, float dc,
                                                 const LstmChildIn& in) {
  const int h = D.h, N = D.N, G = 3 + N;
  const float tc = act_tanh<OpT>(in.cc);
  const float dzo = dh * tc * in.o * (1.f - in.o);
  const float dcb = dc + dh * in.o * (1.f - tc * tc);
  const float dzi = dcb * in.u * in.i * (1.f - in.i);
  const float dzu = dcb * in.i * (1.f - in.u * in.u);
  OpT* dz = op<OpT>(D.dZ) + (size_t)c * G * h;
  dz[j] = to_op<OpT>(dzi); dz[h + j] = to_op<OpT>(dzo); dz[2 * h + j] = to_op<OpT>(dzu);
#pragma unroll
  for (int k = 0; k < kMaxN; ++k) {
    if (k >= N) break;
    const float v = k < c_deg ? dcb * in.ck[k] * in.f[k] * (1.f - in.f[k]) : 0.f;
    dz[(3 + k) * h + j] = to_op<OpT>(v);
  }
  D.dcb[(size_t)c * h + j] = dcb;
}

// ---- epilogue kinds ----------------------------------------------------------------
template <int E> struct EpiK;

// Level kernel, t >= 1: acc = (U_i h~, U_o h~, U_u h~, U_f h_1..U_f h_N).
template <> struct EpiK<EPI_LSTM_FWD> {
  struct In { float ck[kMaxN]; float xi, xo, xu, xf; };
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In& in) {
    const int h = D.h, N = D.N;
    const float* ck = D.Ck + (size_t)m.p * N * h;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) in.ck[k] = k < m.deg ? ck[k * h + j] : 0.f;
    in.xi = in.xo = in.xu = in.xf = 0.f;
    if (m.xrow >= 0) {                           // eager pull projection
      const float* xw = D.XW + (size_t)m.p * 4 * h;
      in.xi = xw[j]; in.xo = xw[h + j]; in.xu = xw[2 * h + j]; in.xf = xw[3 * h + j];
    }
  }
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In& in,
                                               const UnitC& b) {
    float zf[kMaxN];
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) zf[k] = (k < D.N ? acc[3 + k] : 0.f) + in.xf + b.b3;
    lstm_finish<OpT>(D, j, m, acc[0] + in.xi + b.b0, acc[1] + in.xo + b.b1, acc[2] + in.xu + b.b2, zf, in.ck);
  }
};

// Eager pull projection: acc = (W_i x, W_o x, W_u x, W_f x).  Level-0 vertices (no
// children, no recurrent term) are finished here; x-vertices above level 0 keep their
// projection for their own task.
template <> struct EpiK<EPI_LSTM_XPROJ> {
  struct In {};
  static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In&) {}
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In&,
                                               const UnitC& b) {
    const int h = D.h;
    if (m.p < D.lp1) {
      float zf[kMaxN], ck[kMaxN];
#pragma unroll
      for (int k = 0; k < kMaxN; ++k) { zf[k] = acc[3] + b.b3; ck[k] = 0.f; }
      lstm_finish<OpT>(D, j, m, acc[0] + b.b0, acc[1] + b.b1, acc[2] + b.b2, zf, ck);
    } else if (m.xrow >= 0) {
      float* xw = D.XW + (size_t)m.p * 4 * h;
      xw[j] = acc[0]; xw[h + j] = acc[1]; xw[2 * h + j] = acc[2]; xw[3 * h + j] = acc[3];
    }
  }
};

// Backward level epilogue at parent p: acc[0] = U_iou^T dz_iou (= dL/dh~), acc[1+k] = U_f^T dz_fk.
// Gather's adjoint: child k receives dh~ + U_f^T dz_fk (+ its push cotangent) and
// dc-bar * f_k; then dF of the child runs here (the child's own task needs its dZ).
template <> struct EpiK<EPI_LSTM_BWD> {
  struct In { float dcbp; float fp[kMaxN]; LstmChildIn c[kMaxN]; };
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In& in) {
    const int h = D.h, N = D.N;
    in.dcbp = D.dcb[(size_t)m.p * h + j];
    const float* g = D.gates + (size_t)m.p * (3 + N) * h;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) {
      in.fp[k] = k < m.deg ? g[(3 + k) * h + j] : 0.f;
      if (k < m.deg) lstm_child_load(D, j, m.ch[k], m.ch_vid[k], m.ch_deg[k], in.c[k]);
    }
  }
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In& in,
                                               const UnitC&) {
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) {
      if (k >= m.deg) break;
      const float dh = acc[0] + acc[1 + k] + in.c[k].dho;
      lstm_child_store<OpT>(D, j, m.ch[k], m.ch_deg[k], dh, in.dcbp * in.fp[k], in.c[k]);
    }
  }
};

// ---- Tree-FC ------------------------------------------------------------------------
template <class OpT>
__device__ __forceinline__ void fc_finish(const Dev& D, int j, const VMeta& m, float z) {
  const int h = D.h;
  const float hv = act_tanh<OpT>(z);
  D.gates[(size_t)m.p * h + j] = hv;
  D.h_out[(size_t)m.vid * h + j] = hv;
  if (m.par >= 0) op<OpT>(D.Hk)[(size_t)m.par * 2 * h + (size_t)m.slot * h + j] = to_op<OpT>(hv);
}

template <> struct EpiK<EPI_FC_FWD> {
  struct In { float xw; };
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In& in) {
    in.xw = m.xrow >= 0 ? D.XW[(size_t)m.p * D.h + j] : 0.f;
  }
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In& in,
                                               const UnitC& b) {
    fc_finish<OpT>(D, j, m, acc[0] + in.xw + b.b0);
  }
};

template <> struct EpiK<EPI_FC_XPROJ> {
  struct In {};
  static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In&) {}
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In&,
                                               const UnitC& b) {
    if (m.p < D.lp1) fc_finish<OpT>(D, j, m, acc[0] + b.b0);
    else if (m.xrow >= 0) D.XW[(size_t)m.p * D.h + j] = acc[0];
  }
};

// acc[k] = W_{l|r}^T dz  (k = 0: left, 1: right); dz_child = (acc[k] + push cotangent) * (1 - h^2)
template <> struct EpiK<EPI_FC_BWD> {
  struct In { float dho[2], hc[2]; };
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In& in) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      in.dho[k] = k < m.deg ? D.dh_out[(size_t)m.ch_vid[k] * D.h + j] : 0.f;
      in.hc[k] = k < m.deg ? D.gates[(size_t)m.ch[k] * D.h + j] : 0.f;
    }
  }
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In& in,
                                               const UnitC&) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k >= m.deg) break;
      op<OpT>(D.dZ)[(size_t)m.ch[k] * D.h + j] = to_op<OpT>((acc[k] + in.dho[k]) * (1.f - in.hc[k] * in.hc[k]));
    }
  }
};

// pull's adjoint: dx[record] = W^T dz
template <> struct EpiK<EPI_DX> {
  struct In {};
  static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In&) {}
  template <class OpT>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const float* acc, const In&,
                                               const UnitC&) {
    if (m.xrow >= 0) D.dx[(size_t)m.xrow * D.d + j] = acc[0];
  }
};

template <int E> __host__ __device__ constexpr bool epi_needs_children() {
  return E == EPI_LSTM_BWD || E == EPI_FC_BWD;
}
template <int E> __host__ __device__ constexpr bool epi_uses_bias() {
  return E == EPI_LSTM_FWD || E == EPI_LSTM_XPROJ || E == EPI_FC_FWD || E == EPI_FC_XPROJ;
}
template <int E> __host__ __device__ constexpr bool epi_is_lstm() {
  return E == EPI_LSTM_FWD || E == EPI_LSTM_XPROJ || E == EPI_LSTM_BWD;
}

// Does position p need this epilogue at all? (tile skipping for the x-kernels)
template <int E>
__device__ __forceinline__ bool row_active(const Dev& D, int p, int xrow) {
  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ) return p < D.lp1 || xrow >= 0;
  else if constexpr (E == EPI_DX) return xrow >= 0;
  else return true;
}

// dF entry at vertices without a parent: only push's adjoint arrives (dh = Gamma, dc = 0).
template <class OpT>
__device__ __forceinline__ void root_bwd(const Dev& D, int j, int p) {
  const int vid = D.order[p];
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    LstmChildIn in;
    const int deg = D.deg[p];
    lstm_child_load(D, j, p, vid, deg, in);
    lstm_child_store<OpT>(D, j, p, deg, in.dho, 0.f, in);
  } else {
    const float hv = D.gates[(size_t)p * D.h + j];
    op<OpT>(D.dZ)[(size_t)p * D.h + j] = to_op<OpT>(D.dh_out[(size_t)vid * D.h + j] * (1.f - hv * hv));
  }
}

}  // namespace cavs
