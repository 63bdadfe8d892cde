// tc.cu — BF16 path (temporary: SIMT kernels on bf16 operands; tcgen05 kernels follow).
#include "kernels.h"
#include "tc.h"

namespace cavs {

struct TcState { int dummy; };

cavs_status tc_init(const Dev&, int, TcState** out, std::string*) { *out = new TcState{}; return CAVS_OK; }
void tc_destroy(TcState* tc) { delete tc; }

int tc_forward(Dev& D, TcState*, const std::vector<int>& lp, cudaStream_t s) {
  using OpT = __nv_bfloat16;
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  int n = 0;
  SegListI L{};
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    L.n = 4;
    for (int g = 0; g < 4; ++g) L.s[g] = SegI{D.Wb, d, g * h, B_XP, 0, d, d, g};
    simt_typeI<OpT>(D, EPI_LSTM_XPROJ, L, 0, D.V, h, s); ++n;
    SegListI F{};
    F.n = 3 + N;
    for (int g = 0; g < 3; ++g) F.s[g] = SegI{D.Wa, h, g * h, N >= 2 ? B_HSUM : B_HK, 0, N * h, h, g};
    for (int k = 0; k < N; ++k) F.s[3 + k] = SegI{D.Wa, h, 3 * h, B_HK, k * h, N * h, h, 3 + k};
    for (int t = 1; t < T; ++t) { simt_typeI<OpT>(D, EPI_LSTM_FWD, F, lp[t], lp[t + 1], h, s); ++n; }
  } else {
    L.n = 1;
    L.s[0] = SegI{D.Wb, d, 0, B_XP, 0, d, d, 0};
    simt_typeI<OpT>(D, EPI_FC_XPROJ, L, 0, D.V, h, s); ++n;
    SegListI F{};
    F.n = 1;
    F.s[0] = SegI{D.Wa, 2 * h, 0, B_HK, 0, 2 * h, 2 * h, 0};
    for (int t = 1; t < T; ++t) { simt_typeI<OpT>(D, EPI_FC_FWD, F, lp[t], lp[t + 1], h, s); ++n; }
  }
  return n;
}

int tc_backward(Dev& D, TcState*, const std::vector<int>& lp, cudaStream_t s, int* split) {
  using OpT = __nv_bfloat16;
  const int h = D.h, d = D.d, N = D.N, T = (int)lp.size() - 1;
  const int G = D.cell == CAVS_CELL_TREE_LSTM ? 3 + N : 1;
  int n = 0;
  *split = 1;
  SegListI B{};
  int epi;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    B.n = 1 + N;
    B.s[0] = SegI{D.Wc, 3 * h, 0, B_DZ, 0, G * h, 3 * h, 0};
    for (int k = 0; k < N; ++k) B.s[1 + k] = SegI{D.Wd, h, 0, B_DZ, (3 + k) * h, G * h, h, 1 + k};
    epi = EPI_LSTM_BWD;
  } else {
    B.n = 2;
    for (int k = 0; k < 2; ++k) B.s[k] = SegI{D.Wc, h, k * h, B_DZ, 0, h, h, k};
    epi = EPI_FC_BWD;
  }
  for (int t = T - 1; t >= 1; --t) { simt_typeI<OpT>(D, epi, B, lp[t], lp[t + 1], h, s); ++n; }
  float* lz = D.lazy;
  const int lp1 = D.lp1, V = D.V;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    float* u4 = lz; float* uf = u4 + (size_t)3 * h * h; float* w = uf + (size_t)h * h;
    SegListII A{}; A.n = 1;
    A.s[0] = SegII{D.dZ, G * h, 0, N >= 2 ? D.Hs : D.Hk, N >= 2 ? h : N * h, 0, lp1, V, 0};
    simt_typeII<OpT>(D, A, u4, 3 * h, h, h, s);
    SegListII Bf{}; Bf.n = N;
    for (int k = 0; k < N; ++k) Bf.s[k] = SegII{D.dZ, G * h, (3 + k) * h, D.Hk, N * h, k * h, lp1, V, 0};
    simt_typeII<OpT>(D, Bf, uf, h, h, h, s);
    SegListII Cw{}; Cw.n = 1;
    Cw.s[0] = SegII{D.dZ, G * h, 0, D.Xp, d, 0, 0, V, 1};
    simt_typeII<OpT>(D, Cw, w, G * h, d, d, s);
    n += 3;
    SegListI X{}; X.n = 1;
    X.s[0] = SegI{D.We, G * h, 0, B_DZ, 0, G * h, G * h, 0};
    if (D.dx) { simt_typeI<OpT>(D, EPI_DX, X, 0, V, d, s); ++n; }
  } else {
    float* wc = lz; float* wx = wc + (size_t)2 * h * h;
    SegListII A{}; A.n = 1;
    A.s[0] = SegII{D.dZ, h, 0, D.Hk, 2 * h, 0, lp1, V, 0};
    simt_typeII<OpT>(D, A, wc, h, 2 * h, 2 * h, s);
    SegListII Cw{}; Cw.n = 1;
    Cw.s[0] = SegII{D.dZ, h, 0, D.Xp, d, 0, 0, V, 1};
    simt_typeII<OpT>(D, Cw, wx, h, d, d, s);
    n += 2;
    SegListI X{}; X.n = 1;
    X.s[0] = SegI{D.We, h, 0, B_DZ, 0, h, h, 0};
    if (D.dx) { simt_typeI<OpT>(D, EPI_DX, X, 0, V, d, s); ++n; }
  }
  return n;
}

}  // namespace cavs
