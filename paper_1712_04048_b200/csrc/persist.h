// persist.h — persistent weight-stationary level kernels (BF16 mode), see persist.cu.
#pragma once
#include <string>

#include "kernels.h"

namespace cavs {

struct PersistState;
// nullptr (+ reason) when the shape / device does not admit the persistent path.
PersistState* persist_init(const Dev& D, int max_vertices, std::string* why);
void persist_destroy(PersistState* ps);
// clusters (graph ranges) of the persistent kernels: Dev::ncl, the width of the Dev::crow table
int persist_clusters(const PersistState* ps);
// the backward runs the (opt-in) K-split kernel, which takes its task count from the host
bool persist_has_kbwd(const PersistState* ps);
// All tasks t = 1 .. T-1 (forward) / T-1 .. 1 (backward) in one launch.
void persist_forward(const Dev& D, PersistState* ps, int T, cudaStream_t s);
void persist_backward(const Dev& D, PersistState* ps, int T, cudaStream_t s);
// Tree-LSTM backward, K-split with a DSMEM reduction (persist_bwd.cu); nullptr (+ reason) when
// the shape does not admit it.  *clusters: how many clusters of its size can be resident.
struct PbwdState;
PbwdState* pbwd_init(const Dev& D, int max_vertices, int* clusters, std::string* why);
void pbwd_set_clusters(PbwdState* st, int R);
void pbwd_launch(const Dev& D, const PbwdState* st, int T, cudaStream_t s);
void pbwd_destroy(PbwdState* st);
std::string pbwd_describe(const PbwdState* st);
// short description of the plan ("R=9 nub=16 S=3 ...")
std::string persist_describe(const PersistState* ps);

}  // namespace cavs
