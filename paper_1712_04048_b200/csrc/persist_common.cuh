// persist_common.cuh — device helpers shared by the persistent level kernels (persist.cu,
// persist_bwd.cu): suspended mbarrier waits with a trap-on-hang guard, the cluster-local task
// barrier, the per-cluster row table, the SW128 K-major descriptor and the debug trace ring.
#pragma once
#include "cells.cuh"
#include "ptx.cuh"

namespace cavs {

// mbarrier wait: try_wait (the waiting thread is suspended in hardware instead of polling the
// barrier unit), trapping after ~4 s instead of hanging the GPU on a protocol bug.
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  unsigned long long t0 = 0;
  for (;;) {
    uint32_t ok;
#ifdef CAVS_PWAIT_SPIN
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
#endif
    if (ok) return;
    const unsigned long long now = gtime();
    if (t0 == 0) t0 = now;
    else if (now - t0 > 4000000000ull) __trap();
  }
}
// one waiting lane per warp, then the warp proceeds together
__device__ __forceinline__ void pwait_warp(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) pwait(bar, parity);
  __syncwarp();
}

__device__ __forceinline__ int nt_index(int M, int R, int max_ni) {
  const int n = (M + R - 1) / R;
  return min(max_ni, n <= 16 ? 0 : n <= 32 ? 1 : 2);
}

// Cluster-local task barrier.  The graphs of a batch are independent, so each
// cluster owns a contiguous range of graphs (their rows of every task V_t are contiguous: positions
// inside a task are graph-major) and only its own CTAs -- the unit blocks of the same rows -- need
// to agree that V_t is done before V_t+-1 starts.  One mbarrier per CTA counts one remote arrival
// per CTA of the cluster (DSMEM, release at cluster scope); the waiter acquires at cluster scope.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// release-arrive on CTA c's barrier (the release covers this CTA's task writes: the caller passed
// a CTA barrier after them)
__device__ __forceinline__ void cluster_arrive(uint64_t* bar, int c) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(ptx::smem_u32(bar)), "r"(c));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void cluster_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  unsigned long long t0 = 0;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
#ifdef CAVS_PWAIT_SPIN
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
#else
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
#endif
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    const unsigned long long now = gtime();
    if (t0 == 0) t0 = now;
    else if (now - t0 > 4000000000ull) __trap();
  }
}
// rows of task t owned by cluster r: [crow[t][r], crow[t][r + 1]) (k_build_maps)
__device__ __forceinline__ void cl_rows(const Dev& D, int t, int r, int& lo, int& M) {
  const int* c = D.crow + (size_t)t * (D.ncl + 1) + r;
  lo = c[0];
  M = c[1] - lo;
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t lo) {
  return ((uint64_t)((1024u >> 4) | (1u << 14) | (2u << 29)) << 32) | lo;   // SBO 1024, version 1, SWIZZLE_128B
}
// debug trace record (CAVS_TRACE=1): 8 words per record in the ring at D.trace
__device__ __forceinline__ void ptrace(const Dev& D, unsigned long long a, unsigned long long b, unsigned long long c,
                                       unsigned long long d, unsigned long long e, unsigned long long f,
                                       unsigned long long g, unsigned long long h) {
  const unsigned long long at = 8 + 8 * atomicAdd(D.trace, 1ull);
  if (at + 8 < (4u << 20) / 8) {
    D.trace[at] = a; D.trace[at + 1] = b; D.trace[at + 2] = c; D.trace[at + 3] = d;
    D.trace[at + 4] = e; D.trace[at + 5] = f; D.trace[at + 6] = g; D.trace[at + 7] = h;
  }
}


// gate between the epilogue warps (writer: after the cluster task barrier) and the producer /
// epilogue warps of the same CTA: release / acquire at CTA scope
__device__ __forceinline__ void gate_set(int* g, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(ptx::smem_u32(g)), "r"(v) : "memory");
}
__device__ __forceinline__ int gate_get(const int* g) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(g)) : "memory");
  return v;
}

}  // namespace cavs
