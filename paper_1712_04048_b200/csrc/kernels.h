// kernels.h — internal launcher declarations (host side of the engine).
#pragma once
#include <vector>

#include "common.cuh"

namespace cavs {

constexpr int kMaxN = 4;          // max arity supported by the kernels
constexpr int kDbChunks = 32;     // row chunks of the deterministic db column reduction
constexpr int kSplitMax = 8;      // max split-K of the lazy tensor-core GEMMs
constexpr int kLazyMaxTiles = 1024;   // arrival counters of the stream-K lazy kernel (lazy.cu)
constexpr int kMaxClusters = 16;     // graph-range clusters of the persistent level kernels (persist.cu)
constexpr int kDbMaxBlocks = 64;      // arrival counters of the db column blocks (k_colsum)
constexpr int kSkinnyMax = 8;     // tasks with at most this many vertices use the skinny level kernel

enum Epi : int { EPI_LSTM_FWD = 0, EPI_LSTM_XPROJ, EPI_LSTM_BWD, EPI_FC_FWD, EPI_FC_XPROJ, EPI_FC_BWD, EPI_DX,
                 EPI_LSTM_BWD_DAG, EPI_FC_BWD_DAG,
                 EPI_LSTM_FWD_INF, EPI_FC_FWD_INF };   // inference-only forward: no activations for dF
// the training kind an inference kind computes like (same accumulators, same plan)
__host__ __device__ constexpr int epi_base(int E) {
  return E == EPI_LSTM_FWD_INF ? EPI_LSTM_FWD : E == EPI_FC_FWD_INF ? EPI_FC_FWD : E;
}

enum BSrc : int { B_HK = 0, B_XP = 1, B_DZ = 2 };

// One type-I segment: acc[acc] += A[a_row + j, 0:klen] . B[p, b_col : b_col+klen]
struct SegI {
  const void* A; int lda; int a_row;
  int b_src; int b_col; int ldb;
  int klen; int acc;
};
struct SegListI { int n; SegI s[16]; };

// One type-II segment: out[m, n] += sum_{q in [k_lo,k_hi)} A[q, a_col+m] * B[q, b_col+n]
struct SegII {
  const void* A; int lda; int a_col;
  const void* B; int ldb; int b_col;
  int k_lo, k_hi; int skip_no_x;
};
struct SegListII { int n; SegII s[4]; };

// Lazy fp32 scratch: kSplitMax partial slots per GEMM output (float offsets into D.lazy).
struct LazyLayout { size_t u4, uf, w, su4, suf, sw; };
inline LazyLayout lazy_layout(const Dev& D) {
  const size_t h = D.h, d = D.d;
  LazyLayout L{};
  if (D.cell == CAVS_CELL_TREE_LSTM) { L.su4 = 3 * h * h; L.suf = h * h; L.sw = (3 + D.N) * h * d; }
  else { L.su4 = 2 * h * h; L.suf = 0; L.sw = h * d; }
  L.u4 = 0; L.uf = kSplitMax * L.su4; L.w = L.uf + kSplitMax * L.suf;
  return L;
}
inline size_t lazy_floats(const Dev& D) { const LazyLayout L = lazy_layout(D); return L.w + kSplitMax * L.sw; }

// Phase marks (one CUDA event per phase boundary when profiling) + launch counting.
struct Prof {
  bool on = false;
  int cur = -1;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  double ms[CAVS_PH_COUNT] = {}, flops[CAVS_PH_COUNT] = {}, bytes[CAVS_PH_COUNT] = {};
  int64_t launches[CAVS_PH_COUNT] = {};
  int64_t total = 0;
  void mark(int phase, cudaStream_t s) {
    cur = phase;
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    marks.push_back({phase, e});
  }
  void count(int n) { if (cur >= 0) launches[cur] += n; total += n; }
};

// Launch with programmatic dependent launch (PDL): the kernel may be scheduled while its
// predecessor on the stream drains; every such kernel starts with griddepcontrol.wait.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// streaming ablation: the eager x-projection of the tasks above level 0 on a second stream, one
// event per task (owned by the context)
struct XStream { cudaStream_t s = nullptr; std::vector<cudaEvent_t> ev; cudaEvent_t start = nullptr; };

void launch_schedule(const Dev& D, cudaStream_t s);
template <class OpT> void simt_forward(Dev& D, const std::vector<int>& lp, cudaStream_t s, Prof& P,
                                      XStream* xs = nullptr);
template <class OpT> void simt_backward(Dev& D, const std::vector<int>& lp, cudaStream_t s, Prof& P);

template <class OpT>
void simt_typeI(const Dev& D, int epi, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s);
int skinny_max(const Dev& D);   // largest task handled by the skinny kernel (0: unsupported shape)
template <class OpT>
void skinny_typeI(const Dev& D, int epi, const SegListI& L, int row_lo, int row_hi, int units, cudaStream_t s);
// FFMA segment lists of the level kernels (shared by the SIMT, skinny and BF16 paths)
SegListI fwd_segments(const Dev& D);
SegListI bwd_segments(const Dev& D);
template <class OpT>
void simt_typeII(const Dev& D, const SegListII& L, float* out, int M, int Ncols, int ldo, cudaStream_t s,
                 int accum = 0);   // accum: out += (stream-ordered per-task ablation launches)

// ops.cu
void launch_prep(const Dev& D, cudaStream_t s);
void launch_pull(const Dev& D, cudaStream_t s);
void launch_roots(const Dev& D, int n_roots, const int* roots, cudaStream_t s);
void launch_colsum(const Dev& D, float* part, cudaStream_t s);   // db straight into D.dparams
void launch_pack(const Dev& D, const int* split /*[3]*/, cudaStream_t s);   // split-K slots -> dU, dW
// DAG inputs (D.dag): parent CSR of the schedule, the forward gather of task [lo, hi) (children's h, c
// into the parent-slot arenas; fan-out forbids the children's scatter) and the backward pull-reduce
// + dF of task [lo, hi) (sums the edges' gradients in parent-CSR order: deterministic)
// unfused ablation: the cell epilogue `epi` of task rows [lo, hi) from D.raw
void launch_unfused(const Dev& D, int epi, int lo, int hi, cudaStream_t s);
void launch_dag_parents(const Dev& D, cudaStream_t s);
void launch_dx_zero(const Dev& D, cudaStream_t s);   // zero dx unless every record is pulled exactly once
void launch_scatter_rows(float* dst, const float* src, const int* rows, int n, int w, cudaStream_t s);
void launch_dag_gather(const Dev& D, int lo, int hi, cudaStream_t s);
void launch_dag_df(const Dev& D, int lo, int hi, cudaStream_t s);

}  // namespace cavs
