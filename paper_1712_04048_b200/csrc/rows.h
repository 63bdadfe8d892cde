// rows.h — row-tiled tcgen05 level GEMMs for large tasks at h > 512 (fused cell epilogues), see rows.cu.
#pragma once
#include "kernels.h"

namespace cavs {

struct RowsState;
RowsState* rows_init(const Dev& D, int max_vertices);   // nullptr: shape not supported / disabled
void rows_destroy(RowsState* rs);
int rows_tiles(const RowsState* rs, bool backward, int rows);   // size of a task in tiles (or work items, see rows.cu)
int rows_pair(const RowsState* rs);                             // CTAs per MMA (2: cta_group::2 pairs)
// one task V_t = rows [lo, hi) of the forward (or backward) level step; false: caller falls back
bool rows_level(const Dev& D, RowsState* rs, bool backward, int lo, int hi, cudaStream_t s);
// r02: the eager x-projection over all pulled rows / pull's adjoint dX on the row-tiled kernel
// (false: not available for this shape or disabled, CAVS_ROWS_XD=0)
bool rows_xproj(const Dev& D, RowsState* rs, cudaStream_t s);
bool rows_dx(const Dev& D, RowsState* rs, cudaStream_t s);
bool rows_xd(const RowsState* rs);   // the x-projection / dX plans are available

}  // namespace cavs
