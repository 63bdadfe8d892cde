// gemm.h — row-tiled tcgen05 GEMMs with fused cell epilogues (x-projection, dX), see gemm.cu.
#pragma once
#include "kernels.h"

namespace cavs {

struct GemmState;
GemmState* gemm_init(const Dev& D, int max_vertices);   // nullptr: shape not supported / disabled
void gemm_destroy(GemmState* g);
bool gemm_xproj(const Dev& D, GemmState* g, cudaStream_t s);   // false: caller falls back
bool gemm_dx(const Dev& D, GemmState* g, cudaStream_t s);

}  // namespace cavs
