// skinny_f32.cu — FP32 instantiation of the small-task level kernel (skinny.cuh) + its size rule.
#include <cstdlib>

#include "skinny.cuh"

namespace cavs {

int skinny_max(const Dev& D) {
  if (D.split) return 0;   // FP32 split mode: every task runs on the tensor cores (tc.cu)
  static const int env_max = [] {   // CAVS_SKINNY_MAX=n: tasks of <= n vertices on this kernel (0: none)
    const char* e = std::getenv("CAVS_SKINNY_MAX");
    return e ? std::atoi(e) : -1;
  }();
  if (env_max >= 0) return std::min(env_max, kSkinnyMax);
  // h >= 1024 (BF16): the K-sliced gate-split tensor-core kernel beats the FFMA kernel even on tasks of
  // one vertex (cfg4 h = 1024: forward levels 0.564 -> 0.519 ms, profiles/r02_fp32tc.md)
  if (D.prec == CAVS_BF16 && D.h >= 1024) return 0;
  // 16-byte vector access needs every row width / column offset to be a multiple of the vector
  const int es = D.prec == CAVS_BF16 ? 2 : 4;
  const int ve = 16 / es;
  if (D.h % ve || D.d % ve) return 0;
  // staged rows must fit shared memory: widest source row (+ h~) x MV operands
  const int G = D.cell == CAVS_CELL_TREE_LSTM ? 3 + D.N : 1;
  const int W = std::max(D.N * D.h, G * D.h);
  int mv = kSkinnyMax;
  while (mv > 4 && (size_t)mv * W * es > 180 * 1024) mv /= 2;
  return mv;
}

template void skinny_typeI<float>(const Dev&, int, const SegListI&, int, int, int, cudaStream_t);

}  // namespace cavs
