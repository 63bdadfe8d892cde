// sched.cu — on-device scheduler: Algorithm 1's task partition
// and the dynamic-tensor plan (Fig. 7, Alg. 2).
//
// The paper finds activated vertices with a CPU breadth-first search per task
// (P:L396).  Here every graph is swept by one CTA as a parallel frontier sweep
// (indegree countdown): a vertex enters the frontier of round r when its last child
// completed in round r-1, so its round is 1 + max over its children = its task id t
// (reading Z5).  Tasks are then materialised as level-contiguous position lists.
#include <algorithm>

#include "kernels.h"

namespace cavs {

constexpr int kSchedCap = 2048;      // vertices of a graph swept in shared memory (larger: global scratch)

// K1 — one CTA per graph: validation (ranges, arity, fan-out), parents, the frontier sweep
// (level = task id), the graph's level histogram and every vertex's rank among the vertices of
// its graph and level in ascending id (reading Z4).  State lives in shared memory for graphs
// of <= kSchedCap vertices (every BASELINE config), else in the graph's slices of the global
// scratch arrays; local ids throughout.
__global__ void __launch_bounds__(256) k_graph_sched(Dev D) {
  pdl_wait();
  extern __shared__ int sm[];
  const int k = blockIdx.x;
  int* st = D.hdr;
  __shared__ int s_bad, s_head, s_tail;
  const int lo = D.src_gp[k], hi = D.src_gp[k + 1];
  if (threadIdx.x == 0) { s_bad = 0; s_head = 0; s_tail = 0; }
  __syncthreads();
  if (lo < 0 || hi > D.V || hi <= lo || (k == 0 && lo != 0) || (k == D.K - 1 && hi != D.V)) {
    if (threadIdx.x == 0) atomicOr(st, ST_INVALID);
    return;
  }
  const int n = hi - lo;
  // ingest (a1): this graph's slice of the caller's CSR into the workspace copy the later
  // kernels read (a no-op after a host upload, which already wrote the workspace arrays)
  const bool copy = D.src_gp != D.graph_ptr;
  if (copy) {
    if (threadIdx.x == 0) {
      const_cast<int*>(D.graph_ptr)[k] = lo;
      if (k == D.K - 1) const_cast<int*>(D.graph_ptr)[k + 1] = hi;
    }
    for (int i = threadIdx.x; i <= n; i += blockDim.x)
      if (i < n || k == D.K - 1) const_cast<int*>(D.child_ptr)[lo + i] = D.src_cp[lo + i];
    const int e0 = D.src_cp[lo], e1 = D.src_cp[hi];
    if (e0 >= 0 && e1 <= D.E)
      for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) const_cast<int*>(D.child_idx)[e] = D.src_ci[e];
  }
  const bool in_smem = n <= kSchedCap;
  int* par = in_smem ? sm : D.parent_v + lo;                     // local parent id, -1: root
  int* pend = in_smem ? sm + kSchedCap : D.pending + lo;         // children not yet finished
  int* lev = in_smem ? sm + 2 * kSchedCap : D.level + lo;
  int* q = in_smem ? sm + 3 * kSchedCap : D.queue + lo;          // frontier queue (level order)
  int* cnt = in_smem ? sm + 4 * kSchedCap : D.cnt + lo;          // per-level counters (levels < n)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    par[i] = -1;
    cnt[i] = 0;
    D.graph_of[lo + i] = k;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int v = lo + i;
    const int a = D.src_cp[v], b = D.src_cp[v + 1];
    int bad = 0;
    if (a < 0 || b < a || b > D.E) bad |= ST_INVALID;
    else if (b - a > D.N) bad |= ST_ARITY;
    else {
      for (int e = a; e < b; ++e) {
        const int c = D.src_ci[e];
        if (c < 0 || c >= n) { bad |= ST_INVALID; break; }
        if (atomicCAS(&par[c], -1, i) != -1) bad |= ST_FANOUT;
        else D.slot_v[lo + c] = e - a;
      }
    }
    pend[i] = bad ? 0 : b - a;
    if (bad) atomicOr(&s_bad, bad);
  }
  __syncthreads();
  const bool dag = s_bad == ST_FANOUT;               // fan-out only: a DAG (NEXT-3), not an error
  if (s_bad && !dag) {
    if (threadIdx.x == 0) atomicOr(st, s_bad);
    return;
  }
  int round = 0;
  if (dag) {
    // A vertex may have several parents, so there is no single parent to count down: level rounds
    // by pulling instead -- in round r every unassigned vertex whose children all have levels < r
    // gets level r (= 1 + max over its children, reading Z5); no progress with vertices left = cycle.
    if (threadIdx.x == 0) { atomicOr(&st[3], ST_DAG); s_tail = 0; }
    for (int i = threadIdx.x; i < n; i += blockDim.x) lev[i] = -1;
    __syncthreads();
    while (true) {
      __shared__ int s_new;
      if (threadIdx.x == 0) s_new = 0;
      // decide (read every level), then commit (write): no level is read and written in one phase
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        bool ready = lev[i] < 0;
        const int v = lo + i;
        for (int e = D.src_cp[v]; e < D.src_cp[v + 1] && ready; ++e) {
          const int l = lev[D.src_ci[e]];
          ready = l >= 0 && l < round;
        }
        pend[i] = ready ? 1 : 0;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (pend[i]) { lev[i] = round; atomicAdd(&s_new, 1); }
      __syncthreads();
      const int got = s_new;
      __syncthreads();                               // every thread read s_new before its reset
      if (threadIdx.x == 0) s_tail += got;
      if (got == 0) break;
      ++round;
    }
    __syncthreads();
  } else {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (pend[i] == 0) {
      q[atomicAdd(&s_tail, 1)] = i;
      lev[i] = 0;
    }
  }
  __syncthreads();
  while (true) {                                     // round r activates exactly the level-r vertices
    const int qs = s_head, qe = s_tail;
    if (qs == qe) break;
    __syncthreads();
    for (int i = qs + threadIdx.x; i < qe; i += blockDim.x) {
      const int p = par[q[i]];
      if (p >= 0 && atomicSub(&pend[p], 1) == 1) {
        lev[p] = round + 1;
        q[atomicAdd(&s_tail, 1)] = p;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_head = qe;
    ++round;
    __syncthreads();
  }
  }
  if (s_tail != n) {                                 // some vertex never activated
    if (threadIdx.x == 0) atomicOr(st, ST_CYCLE);
    return;
  }
  // ranks inside (graph, level) in ascending id: one warp walks the ids 32 at a time
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int i = b0 + lane;
      const int l = i < n ? lev[i] : -1;
      const unsigned m = __match_any_sync(~0u, l);
      const int leader = __ffs(m) - 1;
      int base = (lane == leader && l >= 0) ? cnt[l] : 0;
      base = __shfl_sync(~0u, base, leader);
      if (i < n) D.lrank[lo + i] = base + __popc(m & ((1u << lane) - 1u));
      __syncwarp();
      if (lane == leader && l >= 0) cnt[l] = base + __popc(m);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (in_smem) D.level[lo + i] = lev[i];
    const int p = par[i];
    D.parent_v[lo + i] = p >= 0 ? lo + p : -1;       // global ids from here on
  }
  if (in_smem)
    for (int l = threadIdx.x; l < round; l += blockDim.x) D.cnt[lo + l] = cnt[l];
  if (threadIdx.x == 0) {
    D.gT[k] = round;                                 // rounds == depth + 1 == this graph's T
    atomicMax(&st[1], round);
  }
}

// Block-wide exclusive scan of one int per thread (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ int block_excl_scan(int x, int* s_warp, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int v = x;
  for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(~0u, v, o); if (lane >= o) v += y; }
  if (lane == 31) s_warp[w] = v;
  __syncthreads();
  if (w == 0) {
    int y = lane < nw ? s_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) { const int z = __shfl_up_sync(~0u, y, o); if (lane >= o) y += z; }
    s_warp[lane] = y;
  }
  __syncthreads();
  total = s_warp[nw - 1];
  const int excl = v - x + (w ? s_warp[w - 1] : 0);
  __syncthreads();
  return excl;
}

// K2 — per task t (CTAs stride over t): exclusive scan over the graphs of their level-t counts
// -> goff[graph_ptr[g] + t] (rows of graph g inside V_t), the task size, and the cluster row
// table of the persistent kernels (crow[t][r] = rows before the first graph of cluster r).  The
// last CTA to finish scans the task sizes into level_ptr and makes crow absolute.
__global__ void __launch_bounds__(1024) k_level_offsets(Dev D) {
  pdl_wait();
  if (D.hdr[0]) return;
  __shared__ int s_warp[32];
  __shared__ int s_last;
  const int T = D.hdr[1], K = D.K, V = D.V, nc = D.ncl;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    int carry = 0;
    for (int g0 = 0; g0 < K; g0 += blockDim.x) {
      const int g = g0 + threadIdx.x;
      const int lo = g < K ? D.graph_ptr[g] : V;
      const bool has = g < K && t < D.gT[g];
      const int c = has ? D.cnt[lo + t] : 0;
      int total;
      const int excl = carry + block_excl_scan(c, s_warp, total);
      if (has) D.goff[lo + t] = excl;
      if (nc > 0 && g < K) {
        const int cg = (int)((long long)lo * nc / V);
        const int cp = g > 0 ? (int)((long long)D.graph_ptr[g - 1] * nc / V) : -1;
        for (int r = cp + 1; r <= cg; ++r) D.crow[(size_t)t * (nc + 1) + r] = excl;
      }
      carry += total;
    }
    if (threadIdx.x == 0) {
      D.lcount[t] = carry;
      if (nc > 0) {
        const int cl = (int)((long long)D.graph_ptr[K - 1] * nc / V);
        for (int r = cl + 1; r <= nc; ++r) D.crow[(size_t)t * (nc + 1) + r] = carry;
      }
    }
  }
  __threadfence();
  __syncthreads();
  int* done = D.tile_cnt + kLazyMaxTiles + kDbMaxBlocks;
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  int carry = 0;
  for (int t0 = 0; t0 < T; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    const int c = t < T ? __ldcg(D.lcount + t) : 0;
    int total;
    const int excl = carry + block_excl_scan(c, s_warp, total);
    if (t < T) D.level_ptr[t] = excl;
    carry += total;
  }
  if (threadIdx.x == 0) { D.level_ptr[T] = V; *done = 0; }
  __syncthreads();
  if (nc > 0)
    for (int i = threadIdx.x; i < T * (nc + 1); i += blockDim.x) {
      const size_t at = i;
      D.crow[at] = __ldcg(D.crow + at) + D.level_ptr[i / (nc + 1)];
    }
}

__device__ __forceinline__ int vpos(const Dev& D, int v, int lo) {
  const int l = D.level[v];
  return D.level_ptr[l] + D.goff[lo + l] + D.lrank[v];
}

// Per vertex: position-indexed plan (children/parent slots, degree).
// K3 — per vertex: position (level_ptr + rows of earlier graphs in the task + rank), order, and
// the position-indexed plan (children / parent slots, degree, roots).
template <class OpT>
__global__ void k_build_maps(Dev D) {
  pdl_wait();
  if (D.hdr[0]) return;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < D.V; v += gridDim.x * blockDim.x) {
    const int lo = D.graph_ptr[D.graph_of[v]];
    const int p = vpos(D, v, lo);
    D.pos[v] = p;
    D.order[p] = v;
    const int a = D.child_ptr[v], deg = D.child_ptr[v + 1] - a;
    D.deg[p] = deg;
    for (int k = 0; k < D.N; ++k)
      D.child_pos[(size_t)p * D.N + k] = k < deg ? vpos(D, lo + D.child_idx[a + k], lo) : -1;
    // DAG batches (fan-out anywhere): no child scatters into a parent slot (the forward gathers
    // per task, launch_dag_gather) and the backward pulls over the parent CSR (launch_dag_df)
    const int pv = (D.hdr[3] & ST_DAG) ? -1 : D.parent_v[v];
    D.parent_pos[p] = pv >= 0 ? vpos(D, pv, lo) : -1;
    D.slot[p] = pv >= 0 ? D.slot_v[v] : 0;
    if (pv < 0) D.roots[atomicAdd(&D.hdr[2], 1)] = p;
    // an internal vertex with fewer than N children reads zero in its missing slots (Z1)
    if (deg > 0 && deg < D.N) {
      OpT* hk = reinterpret_cast<OpT*>(D.Hk) + (size_t)p * D.N * D.h;
      for (int i = deg * D.h; i < D.N * D.h; ++i) st_op1<OpT>(hk + i, 0.f, D.ps_hk);
      if (D.Ck) for (int i = deg * D.h; i < D.N * D.h; ++i) D.Ck[(size_t)p * D.N * D.h + i] = 0.f;
    }
  }
}

void launch_schedule(const Dev& D, cudaStream_t s) {
  static bool attr[kMaxDev] = {};
  constexpr int smem = 5 * kSchedCap * 4;
  const int dv = cur_device();
  if (!attr[dv]) {
    cudaFuncSetAttribute(k_graph_sched, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr[dv] = true;
  }
  launch_pdl(k_graph_sched, dim3(D.K), dim3(256), smem, s, D);
  launch_pdl(k_level_offsets, dim3(148), dim3(1024), 0, s, D);
  const int g = std::min(cdiv(D.V, 256), 148 * 8);
  if (D.prec == CAVS_BF16) launch_pdl(k_build_maps<__nv_bfloat16>, dim3(g), dim3(256), 0, s, D);
  else if (D.split) launch_pdl(k_build_maps<S3>, dim3(g), dim3(256), 0, s, D);
  else launch_pdl(k_build_maps<float>, dim3(g), dim3(256), 0, s, D);
}

}  // namespace cavs
