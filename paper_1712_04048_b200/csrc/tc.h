// tc.h — BF16 tensor-core (tcgen05 + TMA) path of the level kernels and lazy GEMMs.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace cavs {

struct TcState;

cavs_status tc_init(const Dev& D, int max_vertices, TcState** out, std::string* err);
// Returns the number of kernels launched.
int tc_forward(Dev& D, TcState* tc, const std::vector<int>& lp, cudaStream_t s);
int tc_backward(Dev& D, TcState* tc, const std::vector<int>& lp, cudaStream_t s, int* split /*[3]*/);
void tc_destroy(TcState* tc);

}  // namespace cavs
