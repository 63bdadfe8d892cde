// skinny_bf16.cu — BF16 instantiation of the small-task level kernel (skinny.cuh).
#include "skinny.cuh"

namespace cavs {

template void skinny_typeI<__nv_bfloat16>(const Dev&, int, const SegListI&, int, int, int, cudaStream_t);

}  // namespace cavs
