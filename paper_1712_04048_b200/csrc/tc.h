// tc.h — BF16 tensor-core (tcgen05 + TMA) path of the level kernels and lazy GEMMs.
#pragma once
#include <string>
#include <vector>

#include "kernels.h"

namespace cavs {

struct TcState;

cavs_status tc_init(const Dev& D, int max_vertices, TcState** out, std::string* err);
// Launches are counted into P; phase marks XPROJ -> FWD_LEVELS and BWD_LEVELS -> LAZY -> DX.
void tc_forward(Dev& D, TcState* tc, const std::vector<int>& lp, cudaStream_t s, Prof& P, XStream* xs = nullptr);
// the 64 dZ rows past V read by the lazy GEMMs' last k-block -> 0 (any time between the last backward's
// lazy GEMMs and the next one's: cavs_forward issues it beside the pull)
void tc_zero_dz_tail(const Dev& D, const TcState* tc, cudaStream_t s);
// wgrad_ev (nullable): recorded on s once the lazy GEMMs wrote every weight block of dparams
// (stream-K path; otherwise the caller records it after the split-K pack).
void tc_backward(Dev& D, TcState* tc, const std::vector<int>& lp, cudaStream_t s, int* split /*[3]*/, Prof& P,
                 cudaEvent_t wgrad_ev = nullptr, cudaEvent_t levels_ev = nullptr, cudaStream_t dx_s = nullptr);
// levels_ev (nullable): recorded on s once the level tasks wrote every dZ row (db can start)
// dx_s (nullable, needs levels_ev): dX = dZ W runs there, beside the lazy weight-gradient GEMMs on s
void tc_destroy(TcState* tc);
std::string tc_describe(const TcState* tc);   // which level-kernel path is active
int tc_clusters(const TcState* tc);           // graph-range clusters of the persistent level kernels (0: none)
// the whole step runs without host knowledge of the schedule: persistent level kernels (device task
// count), stream-K lazy kernel (device row count), row GEMMs -- the sync-free mode's requirement
bool tc_sync_free_capable(const TcState* tc);

}  // namespace cavs
