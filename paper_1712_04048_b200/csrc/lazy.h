// lazy.h — lazily batched parameter gradients (§3.5 "Lazy batching") as ONE
// stream-K tcgen05 launch with a deterministic in-kernel split-K reduction, see lazy.cu.
#pragma once
#include "kernels.h"

namespace cavs {

struct LazyState;
LazyState* lazy_init(const Dev& D, int max_vertices);   // nullptr: shape not supported / disabled
void lazy_destroy(LazyState* l);
// dU, dW (all blocks) straight into D.dparams (packed layout, OVERWRITTEN); false: caller falls back
bool lazy_grads(const Dev& D, LazyState* l, cudaStream_t s);

}  // namespace cavs
