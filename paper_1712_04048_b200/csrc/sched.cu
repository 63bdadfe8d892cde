// sched.cu — on-device scheduler: Algorithm 1's task partition
// and the dynamic-tensor plan (Fig. 7, Alg. 2).
//
// The paper finds activated vertices with a CPU breadth-first search per task
// (P:L396).  Here every graph is swept by one CTA as a parallel frontier sweep
// (indegree countdown): a vertex enters the frontier of round r when its last child
// completed in round r-1, so its round is 1 + max over its children = its task id t
// (reading Z5).  Tasks are then materialised as level-contiguous position lists.
#include <algorithm>

#include "common.cuh"

namespace cavs {

// One CTA per graph.  Validates (ranges, arity, fan-out), records parents, sweeps.
__global__ void k_graph_levels(Dev D) {
  const int k = blockIdx.x;
  int* st = D.hdr;
  __shared__ int s_bad, s_head, s_tail, s_done, s_round;
  const int lo = D.graph_ptr[k], hi = D.graph_ptr[k + 1];
  if (threadIdx.x == 0) { s_bad = 0; s_head = 0; s_tail = 0; s_done = 0; s_round = 0; }
  __syncthreads();
  if (lo < 0 || hi > D.V || hi <= lo || (k == 0 && lo != 0) || (k == D.K - 1 && hi != D.V)) {
    if (threadIdx.x == 0) atomicOr(st, ST_INVALID);
    return;
  }
  const int n = hi - lo;
  // pass 1: degrees, arity, child ranges; parents (fan-out check)
  for (int v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    D.parent_v[v] = -1;
    D.graph_of[v] = k;
  }
  __syncthreads();
  for (int v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    const int a = D.child_ptr[v], b = D.child_ptr[v + 1];
    int bad = 0;
    if (a < 0 || b < a || b > D.E) bad |= ST_INVALID;
    else if (b - a > D.N) bad |= ST_ARITY;
    else {
      for (int e = a; e < b; ++e) {
        const int c = D.child_idx[e];
        if (c < 0 || c >= n) { bad |= ST_INVALID; break; }
        if (atomicCAS(&D.parent_v[lo + c], -1, v) != -1) bad |= ST_FANOUT;
        else D.slot_v[lo + c] = e - a;
      }
    }
    D.pending[v] = (bad ? 0 : b - a);
    if (bad) { atomicOr(&s_bad, bad); }
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) atomicOr(st, s_bad);
    return;
  }
  // frontier sweep: queue lives in the graph's own slice [lo, hi) of D.queue
  int* q = D.queue + lo;
  for (int v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    if (D.pending[v] == 0) {
      const int at = atomicAdd(&s_tail, 1);
      q[at] = v;
      D.level[v] = 0;
    }
  }
  __syncthreads();
  int round = 0;
  while (true) {
    const int qs = s_head, qe = s_tail;
    if (qs == qe) break;
    __syncthreads();
    for (int i = qs + threadIdx.x; i < qe; i += blockDim.x) {
      const int v = q[i];
      const int p = D.parent_v[v];
      if (p >= 0 && atomicSub(&D.pending[p], 1) == 1) {
        D.level[p] = round + 1;
        const int at = atomicAdd(&s_tail, 1);
        q[at] = p;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_head = qe;
    ++round;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (s_tail != n) atomicOr(st, ST_CYCLE);      // some vertex never activated
    else atomicMax(&st[1], round);               // rounds == depth + 1 == this graph's T
  }
}

__global__ void k_level_hist(Dev D) {
  if (D.hdr[0]) return;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < D.V; v += gridDim.x * blockDim.x)
    atomicAdd(&D.cnt[D.level[v]], 1);
}

// Single CTA: exclusive scan of the level histogram -> level_ptr[0..T].
__global__ void k_level_scan(Dev D) {
  if (D.hdr[0]) return;
  const int T = D.hdr[1];
  __shared__ int s_warp[32];
  __shared__ int s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < T; base += blockDim.x) {
    const int l = base + threadIdx.x;
    const int c = l < T ? D.cnt[l] : 0;
    int x = c;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(~0u, x, o); if (lane >= o) x += y; }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
      int y = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) { int z = __shfl_up_sync(~0u, y, o); if (lane >= o) y += z; }
      s_warp[lane] = y;
    }
    __syncthreads();
    const int incl = x + (w ? s_warp[w - 1] : 0) + s_carry;
    if (l < T) D.level_ptr[l] = incl - c;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) D.level_ptr[T] = D.V;
}

// CTAs stride over levels; each ranks its level's vertices by ascending global id
// (reading Z4) with a block-wide ballot scan over all V vertices.
__global__ void k_level_rank(Dev D) {
  if (D.hdr[0]) return;
  const int T = D.hdr[1];
  __shared__ int s_warp[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = blockIdx.x; l < T; l += gridDim.x) {
    int running = D.level_ptr[l];
    for (int base = 0; base < D.V; base += blockDim.x) {
      const int v = base + threadIdx.x;
      const bool f = v < D.V && D.level[v] == l;
      const unsigned m = __ballot_sync(~0u, f);
      if (lane == 0) s_warp[w] = __popc(m);
      __syncthreads();
      int before = 0, total = 0;
      for (int i = 0; i < nw; ++i) { const int c = s_warp[i]; if (i < w) before += c; total += c; }
      if (f) {
        const int p = running + before + __popc(m & ((1u << lane) - 1));
        D.pos[v] = p;
        D.order[p] = v;
      }
      running += total;
      __syncthreads();
    }
  }
}

// Per vertex: position-indexed plan (children/parent slots, degree).
template <class OpT>
__global__ void k_build_maps(Dev D) {
  if (D.hdr[0]) return;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < D.V; v += gridDim.x * blockDim.x) {
    const int p = D.pos[v];
    const int lo = D.graph_ptr[D.graph_of[v]];
    const int a = D.child_ptr[v], deg = D.child_ptr[v + 1] - a;
    D.deg[p] = deg;
    for (int k = 0; k < D.N; ++k)
      D.child_pos[(size_t)p * D.N + k] = k < deg ? D.pos[lo + D.child_idx[a + k]] : -1;
    const int pv = D.parent_v[v];
    D.parent_pos[p] = pv >= 0 ? D.pos[pv] : -1;
    D.slot[p] = pv >= 0 ? D.slot_v[v] : 0;
    if (pv < 0) D.roots[atomicAdd(&D.hdr[2], 1)] = p;
    if (D.ncl > 0) {
      // graph range of a cluster: cl(g) = graph_ptr[g] * ncl / V (balanced by vertices, monotone
      // in g); inside task t positions are graph-major, so cluster r owns the contiguous rows
      // [crow[t][r], crow[t][r + 1]).  Each entry is written by exactly one vertex: the first of
      // its task whose cluster reaches r, or the task's last vertex for the clusters past it.
      const int t = D.level[v];
      const int t0 = D.level_ptr[t], t1 = D.level_ptr[t + 1];
      const int nc = D.ncl;
      int* row = D.crow + (size_t)t * (nc + 1);
      const int c = (int)((long long)lo * nc / D.V);
      const int cp = p > t0 ? (int)((long long)D.graph_ptr[D.graph_of[D.order[p - 1]]] * nc / D.V) : -1;
      for (int r = cp + 1; r <= c; ++r) row[r] = p;
      if (p == t1 - 1)
        for (int r = c + 1; r <= nc; ++r) row[r] = t1;
    }
    // an internal vertex with fewer than N children reads zero in its missing slots (Z1)
    if (deg > 0 && deg < D.N) {
      OpT* hk = reinterpret_cast<OpT*>(D.Hk) + (size_t)p * D.N * D.h;
      for (int i = deg * D.h; i < D.N * D.h; ++i) hk[i] = to_op<OpT>(0.f);
      if (D.Ck) for (int i = deg * D.h; i < D.N * D.h; ++i) D.Ck[(size_t)p * D.N * D.h + i] = 0.f;
    }
  }
}

void launch_schedule(const Dev& D, cudaStream_t s) {
  k_graph_levels<<<D.K, 256, 0, s>>>(D);
  const int g = std::min(cdiv(D.V, 256), 148 * 8);
  k_level_hist<<<g, 256, 0, s>>>(D);
  k_level_scan<<<1, 1024, 0, s>>>(D);
  k_level_rank<<<148, 1024, 0, s>>>(D);
  if (D.prec == CAVS_BF16) k_build_maps<__nv_bfloat16><<<g, 256, 0, s>>>(D);
  else k_build_maps<float><<<g, 256, 0, s>>>(D);
}

}  // namespace cavs
