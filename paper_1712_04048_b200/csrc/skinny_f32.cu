// skinny_f32.cu — FP32 instantiation of the small-task level kernel (skinny.cuh) + its size rule.
#include "skinny.cuh"

namespace cavs {

int skinny_max(const Dev& D) {
  if (D.split) return 0;   // FP32 split mode: every task runs on the tensor cores (tc.cu)
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
