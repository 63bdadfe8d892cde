// cells.cuh — the vertex function F and its derivative dF as per-(units j..j+VW-1, position p)
// epilogues, shared by every level kernel (FFMA tiles, skinny, tcgen05).
//
// Tree-LSTM, N-ary child-sum (Fig. 5):
//   h~ = sum_k h_k; i = s(W_i x + U_i h~ + b_i); f_k = s(W_f x + U_f h_k + b_f);
//   o = s(W_o x + U_o h~ + b_o); u = tanh(W_u x + U_u h~ + b_u);
//   c = i*u + sum_k f_k*c_k; h = o*tanh(c); scatter [c,h]; push h.
//   (U h~ is accumulated as sum_k U h_k by the GEMMs — the same number in exact arithmetic,
//   reading Z11 of DESIGN.md.)
// Tree-FC (reading Z7): h = tanh(W_c [h_l; h_r] + W_x x + b).
// Backward: hand-derived dF (checked by FD in tests/test_oracle_pins.py);
// gradients flowing to children are written by the unique parent (forests), i.e. the
// "added" of P:L447 is a plain store because every child has exactly one adder.
//
// Every epilogue is split into load() (all global reads of one vertex, into registers) and
// store() (math + all writes), so kernels issue the loads of several vertices before the
// first store: the reads never alias the writes of the same launch (a task's own rows vs.
// its parents' / children's rows).  VW consecutive units are handled per call (VW = 4 in
// the tensor-core kernels: 16-byte accesses); all VW-wide rows are contiguous.
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
// (FP32 mode on tensor cores, OpT = S3, keeps the accurate functions: its parity bar is 1e-5)
template <class OpT> __device__ __forceinline__ float act_sig(float z) {
  if constexpr (sizeof(OpT) == 2 && !is_s3<OpT>::value) return fmaf(0.5f, tanh_fast(0.5f * z), 0.5f);
  else return sigm(z);
}
template <class OpT> __device__ __forceinline__ float act_tanh(float z) {
  if constexpr (sizeof(OpT) == 2 && !is_s3<OpT>::value) return tanh_fast(z);
  else return tanhf(z);
}

// ---- VW-wide vector helpers (VW in {1, 4}) ----------------------------------------------
template <int VW> struct FV { float v[VW]; };

// VW = 8: one 256-bit access per thread (LDG/STG.E.256 on sm_100): a thread that owns one row
// (TMEM lane = vertex, rows.cu) then touches whole 32-byte sectors instead of half sectors.
template <int VW> __device__ __forceinline__ FV<VW> ldv(const float* p) {
  FV<VW> r;
  if constexpr (VW == 8) {
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7]) : "l"(p));
  } else if constexpr (VW == 4) { const float4 t = *reinterpret_cast<const float4*>(p); r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w; }
  else r.v[0] = *p;
  return r;
}
template <int VW> __device__ __forceinline__ void stv(float* p, const FV<VW>& a) {
  if constexpr (VW == 8) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"l"(p), "f"(a.v[0]), "f"(a.v[1]), "f"(a.v[2]), "f"(a.v[3]), "f"(a.v[4]), "f"(a.v[5]), "f"(a.v[6]),
                   "f"(a.v[7]) : "memory");
  } else if constexpr (VW == 4) *reinterpret_cast<float4*>(p) = make_float4(a.v[0], a.v[1], a.v[2], a.v[3]);
  else *p = a.v[0];
}
// ps: plane stride (elements) of the destination arena, used by the split operand type S3 only
template <class OpT, int VW> __device__ __forceinline__ void stv_op(OpT* p, const FV<VW>& a, size_t ps = 0) {
  if constexpr (is_s3<OpT>::value) {
    __nv_bfloat16* q = reinterpret_cast<__nv_bfloat16*>(p);
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      __nv_bfloat16 b0, b1, b2;
      split3(a.v[e], b0, b1, b2);
      q[e] = b0; q[ps + e] = b1; q[2 * ps + e] = b2;
    }
  } else if constexpr (VW == 8 && sizeof(OpT) == 2) {
    uint4 u;
    __nv_bfloat162 b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(a.v[2 * i], a.v[2 * i + 1]);
    u.x = *reinterpret_cast<uint32_t*>(&b[0]); u.y = *reinterpret_cast<uint32_t*>(&b[1]);
    u.z = *reinterpret_cast<uint32_t*>(&b[2]); u.w = *reinterpret_cast<uint32_t*>(&b[3]);
    *reinterpret_cast<uint4*>(p) = u;
  } else if constexpr (VW == 8) {
    stv<8>(reinterpret_cast<float*>(p), a);
  } else if constexpr (VW == 4 && sizeof(OpT) == 2) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a.v[0], a.v[1]), hi = __floats2bfloat162_rn(a.v[2], a.v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(p) = u;
  } else if constexpr (VW == 4) {
    stv<4>(reinterpret_cast<float*>(p), a);
  } else {
    *p = to_op<OpT>(a.v[0]);
  }
}
template <int VW> __device__ __forceinline__ FV<VW> zerov() {
  FV<VW> r;
#pragma unroll
  for (int i = 0; i < VW; ++i) r.v[i] = 0.f;
  return r;
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
template <int VW> struct UnitC { FV<VW> b0, b1, b2, b3; };
template <int VW> __device__ __forceinline__ UnitC<VW> load_unit(const Dev& D, int j, bool lstm) {
  UnitC<VW> u;
  u.b0 = ldv<VW>(D.bias + j);
  if (lstm) { u.b1 = ldv<VW>(D.bias + D.h + j); u.b2 = ldv<VW>(D.bias + 2 * D.h + j); u.b3 = ldv<VW>(D.bias + 3 * D.h + j); }
  else { u.b1 = u.b2 = u.b3 = zerov<VW>(); }
  return u;
}

// ---- Tree-LSTM helpers -----------------------------------------------------------
// Finish F at (j.., p) given gate pre-activations (bias included) and the children's c.
// CHK: 0 = store the activations dF needs; 1 = honour Dev::infer at run time (the x-projection
// epilogue: level-0 cells); 2 = inference kind (EPI_*_FWD_INF: a separate instantiation of the
// level kernels, so the register-bound persistent kernel carries no run-time check).
template <class OpT, int VW, int NM, int CHK = 0>
__device__ __forceinline__ void lstm_finish(const Dev& D, int j, const VMeta& m, const FV<VW>& zi, const FV<VW>& zo,
                                            const FV<VW>& zu, const FV<VW>* zf, const FV<VW>* ck) {
  const bool keep = CHK == 0 || (CHK == 1 && !D.infer);
  const int h = D.h, N = D.N, G = 3 + N;
  FV<VW> i, o, u, c, hv;
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    i.v[e] = act_sig<OpT>(zi.v[e]); o.v[e] = act_sig<OpT>(zo.v[e]); u.v[e] = act_tanh<OpT>(zu.v[e]);
    c.v[e] = i.v[e] * u.v[e];
  }
  float* g = D.gates + (size_t)m.p * G * h + j;
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    if (k >= N) break;
    FV<VW> f;
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      f.v[e] = act_sig<OpT>(zf[k].v[e]);
      if (k < m.deg) c.v[e] = fmaf(f.v[e], ck[k].v[e], c.v[e]);   // missing children: c_k = 0 (Z1)
    }
    if (keep) stv<VW>(g + (3 + k) * h, f);
  }
#pragma unroll
  for (int e = 0; e < VW; ++e) hv.v[e] = o.v[e] * act_tanh<OpT>(c.v[e]);
  if (keep) {                                                       // activations kept for dF
    stv<VW>(g, i); stv<VW>(g + h, o); stv<VW>(g + 2 * h, u);
    stv<VW>(D.cst + (size_t)m.p * h + j, c);
  }
  stv<VW>(D.h_out + (size_t)m.vid * h + j, hv);                   // push(h)
  if (m.par >= 0) {                                                // scatter([c,h]) into the parent's gather slot
    const size_t at = (size_t)m.par * N * h + (size_t)m.slot * h + j;
    stv_op<OpT, VW>(op<OpT>(D.Hk) + at, hv, D.ps_hk);
    stv<VW>(D.Ck + at, c);
  }
}

// dF at child c (units j..): inputs already loaded.
template <int VW, int NM> struct LstmChildIn { FV<VW> dho, i, o, u, cc; FV<VW> f[NM]; FV<VW> ck[NM]; };

template <int VW, int NM>
__device__ __forceinline__ void lstm_child_load(const Dev& D, int j, int c, int c_vid, int c_deg, LstmChildIn<VW, NM>& in) {
  const int h = D.h, N = D.N, G = 3 + N;
  const float* g = D.gates + (size_t)c * G * h + j;
  in.dho = ldv<VW>(D.dh_out + (size_t)c_vid * h + j);
  in.i = ldv<VW>(g); in.o = ldv<VW>(g + h); in.u = ldv<VW>(g + 2 * h);
  in.cc = ldv<VW>(D.cst + (size_t)c * h + j);
  const float* ck = D.Ck + (size_t)c * N * h + j;
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    const bool have = k < c_deg;
    in.f[k] = have ? ldv<VW>(g + (3 + k) * h) : zerov<VW>();
    in.ck[k] = have ? ldv<VW>(ck + k * h) : zerov<VW>();
  }
}

template <class OpT, int VW, int NM>
__device__ __forceinline__ void lstm_child_store(const Dev& D, int j, int c, int c_deg, const FV<VW>& dh,
                                                 const FV<VW>& dc, const LstmChildIn<VW, NM>& in) {
  const int h = D.h, N = D.N, G = 3 + N;
  FV<VW> dzi, dzo, dzu, dcb;
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    const float tc = act_tanh<OpT>(in.cc.v[e]);
    const float o = in.o.v[e], i = in.i.v[e], u = in.u.v[e];
    dzo.v[e] = dh.v[e] * tc * o * (1.f - o);
    dcb.v[e] = dc.v[e] + dh.v[e] * o * (1.f - tc * tc);
    dzi.v[e] = dcb.v[e] * u * i * (1.f - i);
    dzu.v[e] = dcb.v[e] * i * (1.f - u * u);
  }
  OpT* dz = op<OpT>(D.dZ) + (size_t)c * G * h + j;
  stv_op<OpT, VW>(dz, dzi, D.ps_dz); stv_op<OpT, VW>(dz + h, dzo, D.ps_dz); stv_op<OpT, VW>(dz + 2 * h, dzu, D.ps_dz);
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    if (k >= N) break;
    FV<VW> v;
#pragma unroll
    for (int e = 0; e < VW; ++e)
      v.v[e] = k < c_deg ? dcb.v[e] * in.ck[k].v[e] * in.f[k].v[e] * (1.f - in.f[k].v[e]) : 0.f;
    stv_op<OpT, VW>(dz + (3 + k) * h, v, D.ps_dz);
  }
  stv<VW>(D.dcb + (size_t)c * h + j, dcb);
}

// ---- epilogue kinds ----------------------------------------------------------------
template <int E> struct EpiK;

// Level kernel, t >= 1: acc = (U_i h~, U_o h~, U_u h~, U_f h_1..U_f h_N).
template <> struct EpiK<EPI_LSTM_FWD> {
  template <int VW, int NM = kMaxN> struct In { FV<VW> ck[NM]; FV<VW> xi, xo, xu, xf; };
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
    const int h = D.h, N = D.N;
    const float* ck = D.Ck + (size_t)m.p * N * h + j;
#pragma unroll
    for (int k = 0; k < NM; ++k) in.ck[k] = k < m.deg ? ldv<VW>(ck + k * h) : zerov<VW>();
    in.xi = in.xo = in.xu = in.xf = zerov<VW>();
    if (m.xrow >= 0) {                           // eager pull projection
      const float* xw = D.XW + (size_t)m.p * 4 * h + j;
      in.xi = ldv<VW>(xw); in.xo = ldv<VW>(xw + h); in.xu = ldv<VW>(xw + 2 * h); in.xf = ldv<VW>(xw + 3 * h);
    }
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>& b) {
    FV<VW> zi, zo, zu, zf[NM];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      zi.v[e] = acc[0].v[e] + in.xi.v[e] + b.b0.v[e];
      zo.v[e] = acc[1].v[e] + in.xo.v[e] + b.b1.v[e];
      zu.v[e] = acc[2].v[e] + in.xu.v[e] + b.b2.v[e];
    }
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int e = 0; e < VW; ++e) zf[k].v[e] = (k < D.N ? acc[3 + k].v[e] : 0.f) + in.xf.v[e] + b.b3.v[e];
    lstm_finish<OpT, VW, NM>(D, j, m, zi, zo, zu, zf, in.ck);
  }
};

// Eager pull projection: acc = (W_i x, W_o x, W_u x, W_f x).  Level-0 vertices (no
// children, no recurrent term) are finished here; x-vertices above level 0 keep their
// projection for their own task.
template <> struct EpiK<EPI_LSTM_XPROJ> {
  template <int VW, int NM = kMaxN> struct In {};
  template <int VW, int NM = kMaxN> static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In<VW, NM>&) {}
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>&, const UnitC<VW>& b) {
    const int h = D.h;
    if (m.p < dev_lp1(D)) {
      FV<VW> zi, zo, zu, zf[NM], ck[NM];
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        zi.v[e] = acc[0].v[e] + b.b0.v[e]; zo.v[e] = acc[1].v[e] + b.b1.v[e]; zu.v[e] = acc[2].v[e] + b.b2.v[e];
      }
#pragma unroll
      for (int k = 0; k < NM; ++k) {
        ck[k] = zerov<VW>();
#pragma unroll
        for (int e = 0; e < VW; ++e) zf[k].v[e] = acc[3].v[e] + b.b3.v[e];
      }
      lstm_finish<OpT, VW, NM, 1>(D, j, m, zi, zo, zu, zf, ck);
    } else if (m.xrow >= 0) {
      float* xw = D.XW + (size_t)m.p * 4 * h + j;
      stv<VW>(xw, acc[0]); stv<VW>(xw + h, acc[1]); stv<VW>(xw + 2 * h, acc[2]); stv<VW>(xw + 3 * h, acc[3]);
    }
  }
};

// Backward level epilogue at parent p: acc[0] = U_iou^T dz_iou (= dL/dh~), acc[1+k] = U_f^T dz_fk.
// Gather's adjoint: child k receives dh~ + U_f^T dz_fk (+ its push cotangent) and
// dc-bar * f_k; then dF of the child runs here (the child's own task needs its dZ).
template <> struct EpiK<EPI_LSTM_BWD> {
  template <int VW, int NM = kMaxN> struct In { FV<VW> dcbp; FV<VW> fp[NM]; LstmChildIn<VW, NM> c[NM]; };
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
    const int h = D.h, N = D.N;
    in.dcbp = ldv<VW>(D.dcb + (size_t)m.p * h + j);
    const float* g = D.gates + (size_t)m.p * (3 + N) * h + j;
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      in.fp[k] = k < m.deg ? ldv<VW>(g + (3 + k) * h) : zerov<VW>();
      if (k < m.deg) lstm_child_load<VW, NM>(D, j, m.ch[k], m.ch_vid[k], m.ch_deg[k], in.c[k]);
    }
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>&) {
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      if (k >= m.deg) break;
      FV<VW> dh, dc;
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        dh.v[e] = acc[0].v[e] + acc[1 + k].v[e] + in.c[k].dho.v[e];
        dc.v[e] = in.dcbp.v[e] * in.fp[k].v[e];
      }
      lstm_child_store<OpT, VW, NM>(D, j, m.ch[k], m.ch_deg[k], dh, dc, in.c[k]);
    }
  }
};

// ---- Tree-FC ------------------------------------------------------------------------
template <class OpT, int VW, int CHK = 0>
__device__ __forceinline__ void fc_finish(const Dev& D, int j, const VMeta& m, const FV<VW>& z) {
  const int h = D.h;
  FV<VW> hv;
#pragma unroll
  for (int e = 0; e < VW; ++e) hv.v[e] = act_tanh<OpT>(z.v[e]);
  if (CHK == 0 || (CHK == 1 && !D.infer)) stv<VW>(D.gates + (size_t)m.p * h + j, hv);   // h kept for dF (1 - h^2)
  stv<VW>(D.h_out + (size_t)m.vid * h + j, hv);
  if (m.par >= 0) stv_op<OpT, VW>(op<OpT>(D.Hk) + (size_t)m.par * 2 * h + (size_t)m.slot * h + j, hv, D.ps_hk);
}

template <> struct EpiK<EPI_FC_FWD> {
  template <int VW, int NM = kMaxN> struct In { FV<VW> xw; };
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
    in.xw = m.xrow >= 0 ? ldv<VW>(D.XW + (size_t)m.p * D.h + j) : zerov<VW>();
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>& b) {
    FV<VW> z;
#pragma unroll
    for (int e = 0; e < VW; ++e) z.v[e] = acc[0].v[e] + in.xw.v[e] + b.b0.v[e];
    fc_finish<OpT, VW>(D, j, m, z);
  }
};

template <> struct EpiK<EPI_FC_XPROJ> {
  template <int VW, int NM = kMaxN> struct In {};
  template <int VW, int NM = kMaxN> static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In<VW, NM>&) {}
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>&, const UnitC<VW>& b) {
    if (m.p < dev_lp1(D)) {
      FV<VW> z;
#pragma unroll
      for (int e = 0; e < VW; ++e) z.v[e] = acc[0].v[e] + b.b0.v[e];
      fc_finish<OpT, VW, 1>(D, j, m, z);
    } else if (m.xrow >= 0) {
      stv<VW>(D.XW + (size_t)m.p * D.h + j, acc[0]);
    }
  }
};

// Inference-only forward kinds: the training epilogue without the activations dF needs.
template <> struct EpiK<EPI_LSTM_FWD_INF> {
  template <int VW, int NM = kMaxN> using In = EpiK<EPI_LSTM_FWD>::In<VW, NM>;
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
    EpiK<EPI_LSTM_FWD>::load<VW, NM>(D, j, m, in);
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>& b) {
    FV<VW> zi, zo, zu, zf[NM];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      zi.v[e] = acc[0].v[e] + in.xi.v[e] + b.b0.v[e];
      zo.v[e] = acc[1].v[e] + in.xo.v[e] + b.b1.v[e];
      zu.v[e] = acc[2].v[e] + in.xu.v[e] + b.b2.v[e];
    }
#pragma unroll
    for (int k = 0; k < NM; ++k)
#pragma unroll
      for (int e = 0; e < VW; ++e) zf[k].v[e] = (k < D.N ? acc[3 + k].v[e] : 0.f) + in.xf.v[e] + b.b3.v[e];
    lstm_finish<OpT, VW, NM, 2>(D, j, m, zi, zo, zu, zf, in.ck);
  }
};
template <> struct EpiK<EPI_FC_FWD_INF> {
  template <int VW, int NM = kMaxN> using In = EpiK<EPI_FC_FWD>::In<VW, NM>;
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
    EpiK<EPI_FC_FWD>::load<VW, NM>(D, j, m, in);
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>& b) {
    FV<VW> z;
#pragma unroll
    for (int e = 0; e < VW; ++e) z.v[e] = acc[0].v[e] + in.xw.v[e] + b.b0.v[e];
    fc_finish<OpT, VW, 2>(D, j, m, z);
  }
};

// acc[k] = W_{l|r}^T dz  (k = 0: left, 1: right); dz_child = (acc[k] + push cotangent) * (1 - h^2)
template <> struct EpiK<EPI_FC_BWD> {
  template <int VW, int NM = kMaxN> struct In { FV<VW> dho[2], hc[2]; };
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      in.dho[k] = k < m.deg ? ldv<VW>(D.dh_out + (size_t)m.ch_vid[k] * D.h + j) : zerov<VW>();
      in.hc[k] = k < m.deg ? ldv<VW>(D.gates + (size_t)m.ch[k] * D.h + j) : zerov<VW>();
    }
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>&) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k >= m.deg) break;
      FV<VW> dz;
#pragma unroll
      for (int e = 0; e < VW; ++e) dz.v[e] = (acc[k].v[e] + in.dho[k].v[e]) * (1.f - in.hc[k].v[e] * in.hc[k].v[e]);
      stv_op<OpT, VW>(op<OpT>(D.dZ) + (size_t)m.ch[k] * D.h + j, dz, D.ps_dz);
    }
  }
};

// ---- DAG inputs (fan-out): the level GEMM's epilogue only sends the gradient along each edge; the
// child's dF runs once all its parents are done (launch_dag_df: fixed-order sum over its parents).
// Tree-LSTM at parent p, slot k: dL/dh_k = U_iou^T dz_iou + U_f^T dz_fk, dL/dc_k = dc-bar * f_k.
template <> struct EpiK<EPI_LSTM_BWD_DAG> {
  template <int VW, int NM = kMaxN> struct In { FV<VW> dcbp; FV<VW> fp[NM]; };
  template <int VW, int NM = kMaxN>
  static __device__ __forceinline__ void load(const Dev& D, int j, const VMeta& m, In<VW, NM>& in) {
    const int h = D.h, N = D.N;
    in.dcbp = ldv<VW>(D.dcb + (size_t)m.p * h + j);
    const float* g = D.gates + (size_t)m.p * (3 + N) * h + j;
#pragma unroll
    for (int k = 0; k < NM; ++k) in.fp[k] = k < m.deg ? ldv<VW>(g + (3 + k) * h) : zerov<VW>();
  }
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>& in, const UnitC<VW>&) {
    const int h = D.h, N = D.N;
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      if (k >= m.deg) break;
      FV<VW> dh, dc;
#pragma unroll
      for (int e = 0; e < VW; ++e) { dh.v[e] = acc[0].v[e] + acc[1 + k].v[e]; dc.v[e] = in.dcbp.v[e] * in.fp[k].v[e]; }
      const size_t at = ((size_t)m.p * N + k) * h + j;
      stv<VW>(D.dHg + at, dh);
      stv<VW>(D.dCg + at, dc);
    }
  }
};
// Tree-FC at parent p: dL/dh_k = W_k^T dz (acc[k]).
template <> struct EpiK<EPI_FC_BWD_DAG> {
  template <int VW, int NM = kMaxN> struct In {};
  template <int VW, int NM = kMaxN> static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In<VW, NM>&) {}
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>&, const UnitC<VW>&) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (k < m.deg) stv<VW>(D.dHg + ((size_t)m.p * 2 + k) * D.h + j, acc[k]);
  }
};

// pull's adjoint: dx[record] += W^T dz.  ADDED, not stored: several vertices may pull
// the same record (an embedding row); dx is zeroed by cavs_backward first.  With one vertex per
// record every element receives exactly one add onto 0 (deterministic).
template <int VW> __device__ __forceinline__ void addv(float* p, const FV<VW>& a) {
  if constexpr (VW == 8) {
    atomicAdd(reinterpret_cast<float4*>(p), make_float4(a.v[0], a.v[1], a.v[2], a.v[3]));
    atomicAdd(reinterpret_cast<float4*>(p + 4), make_float4(a.v[4], a.v[5], a.v[6], a.v[7]));
  } else if constexpr (VW == 4) {
    atomicAdd(reinterpret_cast<float4*>(p), make_float4(a.v[0], a.v[1], a.v[2], a.v[3]));
  } else {
    atomicAdd(p, a.v[0]);
  }
}
template <> struct EpiK<EPI_DX> {
  template <int VW, int NM = kMaxN> struct In {};
  template <int VW, int NM = kMaxN> static __device__ __forceinline__ void load(const Dev&, int, const VMeta&, In<VW, NM>&) {}
  template <class OpT, int VW, int NM = kMaxN>
  static __device__ __forceinline__ void store(const Dev& D, int j, const VMeta& m, const FV<VW>* acc,
                                               const In<VW, NM>&, const UnitC<VW>&) {
    if (m.xrow < 0) return;
    float* dst = D.dx + (size_t)m.xrow * D.d + j;
    if (D.hdr[5]) addv<VW>(dst, acc[0]);             // a record pulled by several vertices: add
    else stv<VW>(dst, acc[0]);                       // each record pulled at most once: one store
  }
};

template <int E> __host__ __device__ constexpr bool epi_needs_children() {
  return E == EPI_LSTM_BWD || E == EPI_FC_BWD;
}
template <int E> __host__ __device__ constexpr bool epi_uses_bias() {
  return E == EPI_LSTM_FWD || E == EPI_LSTM_XPROJ || E == EPI_FC_FWD || E == EPI_FC_XPROJ || E == EPI_LSTM_FWD_INF ||
         E == EPI_FC_FWD_INF;
}
template <int E> __host__ __device__ constexpr bool epi_is_lstm() {
  return E == EPI_LSTM_FWD || E == EPI_LSTM_XPROJ || E == EPI_LSTM_BWD || E == EPI_LSTM_BWD_DAG || E == EPI_LSTM_FWD_INF;
}

// Does position p need this epilogue at all? (tile skipping for the x-kernels)
template <int E>
__device__ __forceinline__ bool row_active(const Dev& D, int p, int xrow) {
  if constexpr (E == EPI_LSTM_XPROJ || E == EPI_FC_XPROJ) return p < dev_lp1(D) || xrow >= 0;
  else if constexpr (E == EPI_DX) return xrow >= 0;
  else return true;
}

// The level-task epilogues (the ones the unfused ablation splits off the GEMM).
template <int E> __host__ __device__ constexpr bool epi_is_level() {
  return E == EPI_LSTM_FWD || E == EPI_LSTM_BWD || E == EPI_FC_FWD || E == EPI_FC_BWD || E == EPI_LSTM_BWD_DAG ||
         E == EPI_FC_BWD_DAG;
}
// Unfused ablation: the GEMM only stores its accumulators (acc e of unit j at raw[p][e h + j]).
template <int VW>
__device__ __forceinline__ void store_raw(const Dev& D, int j, int p, const FV<VW>* acc, int nacc) {
  for (int e = 0; e < nacc && e * D.h < D.rawld; ++e) stv<VW>(D.raw + (size_t)p * D.rawld + (size_t)e * D.h + j, acc[e]);
}

// Scalar entry used by the FFMA / skinny kernels: acc has NACC entries.
template <int E, class OpT, int NACC>
__device__ __forceinline__ void epilogue1(const Dev& D, int j, const VMeta& m, const float* acc) {
  if constexpr (epi_is_level<E>()) {
    if (D.unfused) {
      for (int e = 0; e < NACC && e * D.h < D.rawld; ++e) D.raw[(size_t)m.p * D.rawld + (size_t)e * D.h + j] = acc[e];
      return;
    }
  }
  const UnitC<1> uc = epi_uses_bias<E>() ? load_unit<1>(D, j, epi_is_lstm<E>()) : UnitC<1>{};
  FV<1> a[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) a[q].v[0] = acc[q];
  typename EpiK<E>::template In<1, kMaxN> in;
  EpiK<E>::template load<1, kMaxN>(D, j, m, in);
  EpiK<E>::template store<OpT, 1, kMaxN>(D, j, m, a, in, uc);
}

// DAG: dF at position p once every parent sent its edge gradients (dHg / dCg at the parent-slot
// indices pent[pptr[p] .. pptr[p+1]), ascending: a fixed summation order), plus push's adjoint.
template <class OpT>
__device__ __forceinline__ void dag_df(const Dev& D, int j, int p) {
  const int vid = D.order[p];
  const int e0 = D.pptr[p], e1 = D.pptr[p + 1];
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    LstmChildIn<1, kMaxN> in;
    const int deg = D.deg[p];
    lstm_child_load<1, kMaxN>(D, j, p, vid, deg, in);
    FV<1> dh = in.dho, dc = zerov<1>();
    for (int e = e0; e < e1; ++e) {
      const size_t at = (size_t)D.pent[e] * D.h + j;
      dh.v[0] += D.dHg[at];
      dc.v[0] += D.dCg[at];
    }
    lstm_child_store<OpT, 1, kMaxN>(D, j, p, deg, dh, dc, in);
  } else {
    float dh = D.dh_out[(size_t)vid * D.h + j];
    for (int e = e0; e < e1; ++e) dh += D.dHg[(size_t)D.pent[e] * D.h + j];
    const float hv = D.gates[(size_t)p * D.h + j];
    st_op1<OpT>(op<OpT>(D.dZ) + (size_t)p * D.h + j, dh * (1.f - hv * hv), D.ps_dz);
  }
}

// dF entry at vertices without a parent: only push's adjoint arrives (dh = Gamma, dc = 0).
template <class OpT>
__device__ __forceinline__ void root_bwd(const Dev& D, int j, int p) {
  const int vid = D.order[p];
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    LstmChildIn<1, kMaxN> in;
    const int deg = D.deg[p];
    lstm_child_load<1, kMaxN>(D, j, p, vid, deg, in);
    lstm_child_store<OpT, 1, kMaxN>(D, j, p, deg, in.dho, zerov<1>(), in);
  } else {
    const float hv = D.gates[(size_t)p * D.h + j];
    st_op1<OpT>(op<OpT>(D.dZ) + (size_t)p * D.h + j, D.dh_out[(size_t)vid * D.h + j] * (1.f - hv * hv), D.ps_dz);
  }
}

}  // namespace cavs
