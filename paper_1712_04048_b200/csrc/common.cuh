// common.cuh — shared device/host definitions of the Cavs B200 engine (internal).
//
// Data layout in HBM: every per-vertex tensor of F is a
// "dynamic tensor" (Fig. 7) laid out in POSITION order: the
// vertices of task V_0 first, then V_1, ..., each task contiguous (offset of task t =
// level_ptr[t] rows, bs = M_t).  Gather buffers are PARENT-slot arenas: a child's
// scatter writes its state straight into row pos(parent), slot k of the gather arena
// (Hk/Ck), so a task's gather operand is a contiguous row block.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/cavs.h"

namespace cavs {

enum : int { ST_INVALID = 1, ST_ARITY = 2, ST_CYCLE = 4, ST_FANOUT = 8, ST_XROW = 16, ST_DAG = 32 };

// Device view of one context: sizes + every arena pointer.  Passed by value.
struct Dev {
  int cell, N, h, d, prec;
  int K, V, E, n_x, T, lp1;          // lp1 = level_ptr[1] (first internal position), host copy
  int infer;                        // 1: inference-only forward (no activations saved for dF)
  // loaded graphs (global CSR, instance-local child ids)
  const int* graph_ptr; const int* child_ptr; const int* child_idx;
  // where k_graph_sched reads the CSR: the caller's device arrays (copied into the arrays above
  // by the same kernel) or, after a host upload, the arrays above themselves
  const int* src_gp; const int* src_cp; const int* src_ci;
  // schedule (vid-indexed)
  int* level; int* pos; int* graph_of; int* parent_v; int* slot_v; int* pending; int* queue;
  // schedule (position-indexed)
  int* order; int* level_ptr; int* child_pos; int* parent_pos; int* slot; int* deg; int* xrow_pos;
  int* tile_x;                      // per 64-position tile: 1 if any vertex has a pull record
  int* hdr;                         // [0] status bits, [1] T, [2] #roots, [3] ST_XROW (deferred input error) | ST_DAG,
                                    // [4] vertices with a record, [5] 1: a record pulled twice (both reset by the
                                    // forward before k_pull), [6..] level_ptr
  int* xseen; unsigned xgen;        // per record: generation of the last forward that pulled it (duplicate pulls)
  int* roots;                       // positions of vertices without a parent
  int* cnt;                         // per-graph level histograms: cnt[graph_ptr[g] + t] (t < T_g)
  int* lrank;                       // rank of a vertex among the vertices of its graph and level
  int* goff;                        // goff[graph_ptr[g] + t]: rows of earlier graphs in task t
  int* gT;                          // levels of graph g
  int* lcount;                      // |V_t|
  unsigned* gsync;                  // [0] barrier arrivals, [1] exits: grid barrier of the persistent level kernels
  int ncl;                          // clusters of the persistent level kernels (0: none)
  int* crow;                        // [T][ncl + 1]: first position of task t owned by cluster >= r
  int* tile_cnt;                    // arrival counters (zero between launches): lazy tiles, then db column blocks
  float* rows_part;                 // split-K partial accumulators of the row-tiled level GEMMs (rows.cu), or null
  int* rows_cnt;                    // their per-tile arrival counters (zero between launches)
  // engine ablations of the paper's optimisations, fixed at
  // cavs_create from the environment: lazy_off (CAVS_LAZY_BATCH=0), unfused
  // (CAVS_UNFUSED=1: the level GEMMs store raw accumulators, a separate elementwise
  // kernel applies F / dF), stream_x (CAVS_STREAMING=1: the eager x-projection of the tasks
  // above level 0 runs on a second stream, each task waiting only for its own rows)
  int lazy_off, unfused, stream_x;
  // sync-free mode (cavs_set_sync_free): the host never reads the schedule header; the kernels
  // take T, level_ptr[1] and #roots from the device header (dev_T / dev_lp1), and skip their work
  // for an invalid or DAG batch (reported by cavs_sync)
  int sync_free;
  float* raw; int rawld;            // unfused: raw accumulators [Vp, rawld] fp32
  // DAG inputs (fan-out: a vertex with several parents); dag = 1 for this batch
  int dag;
  int* pptr;                        // [V+1] parent CSR by position: entries [pptr[p], pptr[p+1])
  int* pent;                        // [E] parent-slot index q = parent_pos * N + k, ascending per vertex
  int* pcur;                        // [V] fill cursors
  float* dHg;                       // [Vp, N*h] gradient sent along edge (parent p, slot k): dL/dh_k
  float* dCg;                       // [Vp, N*h] Tree-LSTM: dL/dc_k along the same edge
  // arenas (OpT = float in FP32 mode, __nv_bfloat16 in BF16 mode)
  void* Hk;      // [Vp, N*h] gather slots of child h (written by the child's scatter)
  void* Hs;      // [Vp, h]   child-sum h~ (Tree-LSTM, N >= 2)
  void* Xp;      // [Vp, d]   pulled x in position order (zero rows: no record)
  void* dZ;      // [Vp, G*h] gate-preactivation gradients (G = 3+N Tree-LSTM, 1 Tree-FC)
  float* Ck;     // [Vp, N*h] gather slots of child c (Tree-LSTM)
  float* XW;     // [Vp, Gx*h] eager x-projection for x-vertices above level 0
  float* gates;  // [Vp, G*h] Tree-LSTM activations (i,o,u,f_1..f_N); Tree-FC: h
  float* cst;    // [Vp, h]   Tree-LSTM memory cell c
  float* dcb;    // [Vp, h]   Tree-LSTM dc-bar
  float* bias;   // internal gate order (i,o,u,f) / (b)
  // weight copies (OpT), see prep kernel
  void* Wa; void* Wb; void* Wc; void* Wd; void* We;
  // lazy outputs (fp32 scratch)
  float* lazy;
  // FP32 mode on tensor cores (bf16x3 split): split = 1 stores every operand
  // arena / weight copy as three bf16 planes x = b0 + b1 + b2; plane q of an arena lives q * ps_*
  // elements after plane 0 (plane-major: the row arithmetic of plane 0 is unchanged)
  int split;
  size_t ps_hk, ps_xp, ps_dz;       // plane strides (elements) of Hk, Xp, dZ
  size_t ps_w[5];                   // plane strides of the weight copies Wa..We
  unsigned long long* trace;   // debug (CAVS_TRACE=1): per-CTA globaltimer records, else null
  // caller buffers of the current call
  const float* params; const float* x; const int* x_row; const float* dh_out;
  float* h_out; float* dparams; float* dx;
};

constexpr int kPadRows = 128;   // extra zero rows after V for TMA/K-block over-reach
constexpr int kHdrWords = 6;    // header words before level_ptr (cavs_api.cu carve)

// Schedule facts on the device (sync-free mode) or from the host copy.  Read after the PDL wait.
__device__ __forceinline__ bool dev_skip(const struct Dev& D);

// cudaFuncSetAttribute is per device: launchers cache "attribute already set" per device id.
constexpr int kMaxDev = 64;
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : d % kMaxDev;
}


__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float sigm(float z) { return 1.0f / (1.0f + expf(-z)); }

template <class T> __device__ __forceinline__ T to_op(float v);
template <> __device__ __forceinline__ float to_op<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 to_op<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
__device__ __forceinline__ float from_op(float v) { return v; }
__device__ __forceinline__ float from_op(__nv_bfloat16 v) { return __bfloat162float(v); }

// Operand type of the FP32-on-tensor-core mode: plane 0 of a bf16x3 split value (the bf16 bits of
// b0 = rn(x); planes 1, 2 hold b1 = rn(x - b0), b2 = rn(x - b0 - b1) one plane stride further).
// Both differences are exact in fp32 (Sterbenz), so b0 + b1 + b2 = x to within 2^-24 |x|, and the
// six products a_s b_t (s + t <= 2) of two split operands give x y to ~2^-22 relative.
struct S3 { __nv_bfloat16 b; };
template <class T> struct is_s3 { static constexpr bool value = false; };
template <> struct is_s3<S3> { static constexpr bool value = true; };
__device__ __forceinline__ void split3(float x, __nv_bfloat16& b0, __nv_bfloat16& b1, __nv_bfloat16& b2) {
  b0 = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(b0);
  b1 = __float2bfloat16_rn(r1);
  b2 = __float2bfloat16_rn(r1 - __bfloat162float(b1));
}
// one operand value: plain store (fp32 / bf16) or the three planes (S3, plane stride ps)
template <class OpT> __device__ __forceinline__ void st_op1(OpT* p, float v, size_t ps) {
  if constexpr (is_s3<OpT>::value) {
    __nv_bfloat16 b0, b1, b2;
    split3(v, b0, b1, b2);
    __nv_bfloat16* q = reinterpret_cast<__nv_bfloat16*>(p);
    q[0] = b0; q[ps] = b1; q[2 * ps] = b2;
  } else {
    (void)ps;
    *p = to_op<OpT>(v);
  }
}
template <class OpT> __device__ __forceinline__ float ld_op1(const OpT* p, size_t ps) {
  if constexpr (is_s3<OpT>::value) {
    const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(p);
    return (__bfloat162float(q[0]) + __bfloat162float(q[ps])) + __bfloat162float(q[2 * ps]);
  } else {
    (void)ps;
    return from_op(*p);
  }
}

__device__ __forceinline__ bool dev_skip(const Dev& D) {
  return D.sync_free && (D.hdr[0] != 0 || (D.hdr[3] & ST_DAG) != 0);
}
__device__ __forceinline__ int dev_T(const Dev& D) { return D.sync_free ? (dev_skip(D) ? 0 : D.hdr[1]) : D.T; }
__device__ __forceinline__ int dev_lp1(const Dev& D) {
  if (!D.sync_free) return D.lp1;
  const int T = dev_T(D);
  return T > 1 ? D.hdr[kHdrWords + 1] : D.V;
}

}  // namespace cavs
