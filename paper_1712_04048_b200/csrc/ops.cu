// ops.cu — small HBM-bound kernels around the level loop:
//   k_prep   : repack fp32 params into the internal gate order / operand dtype (static
//              tensors for parameters), incl. transposed copies for dF's GEMMs;
//   k_pull   : pull() as one batched indexed copy into the position-ordered x arena
//              (Alg. 2's gather/pull memcpy), + per-tile "has x" flags;
//   k_roots  : dF's entry at vertices without a parent (push's adjoint only);
//   k_colsum : deterministic column sums of dZ (db), lazily over all vertices;
//   k_pack   : lazy outputs -> packed dparams (sums split-K partials and the f_k blocks).
#include <algorithm>

#include "cells.cuh"
#include "kernels.h"

namespace cavs {

// Parameter repack as a list of jobs, one launch: blockIdx.y = job.  A copy job converts a
// contiguous fp32 range; a transpose job writes dst[c][r] = src[r][c] (32 x 32 smem tiles, both
// sides coalesced).  The internal layouts are plain concatenations / transposes of the packed
// blocks (internal gate order (i, o, u, f); packed W/b order (i, f, o, u)).
struct PrepJob {
  const float* src; int rows, cols, spitch;    // source block (row-major fp32)
  int dst_sel; size_t dst_off; int dpitch;     // destination arena (0..4: Wa..We, 5: bias fp32)
  int transpose;
};
struct PrepJobs { int n; PrepJob j[20]; };

template <class OpT>
__device__ __forceinline__ OpT* prep_dst(const Dev& D, int sel) {
  return sel == 0 ? op<OpT>(D.Wa) : sel == 1 ? op<OpT>(D.Wb) : sel == 2 ? op<OpT>(D.Wc) : sel == 3 ? op<OpT>(D.Wd)
                                                                                          : op<OpT>(D.We);
}

template <class OpT>
__global__ void __launch_bounds__(256) k_prep(Dev D, PrepJobs J) {
  pdl_wait();
  const PrepJob& jb = J.j[blockIdx.y];
  __shared__ float tile[32][33];
  if (jb.transpose) {
    const int tr = cdiv(jb.rows, 32), tc = cdiv(jb.cols, 32);
    OpT* dst = prep_dst<OpT>(D, jb.dst_sel) + jb.dst_off;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;        // 32 x 8
    for (int t = blockIdx.x; t < tr * tc; t += gridDim.x) {
      const int r0 = (t / tc) * 32, c0 = (t % tc) * 32;
#pragma unroll
      for (int k = 0; k < 32; k += 8) {
        const int r = r0 + ty + k, c = c0 + tx;
        tile[ty + k][tx] = (r < jb.rows && c < jb.cols) ? jb.src[(size_t)r * jb.spitch + c] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 32; k += 8) {
        const int c = c0 + ty + k, r = r0 + tx;                    // dst row = source column
        if (r < jb.rows && c < jb.cols) st_op1<OpT>(dst + (size_t)c * jb.dpitch + r, tile[tx][ty + k], D.ps_w[jb.dst_sel]);
      }
      __syncthreads();
    }
  } else {
    const size_t n = (size_t)jb.rows * jb.cols;                  // contiguous (spitch == cols)
    if (jb.dst_sel == 5) {
      for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        D.bias[jb.dst_off + i] = jb.src[i];
      return;
    }
    OpT* dst = prep_dst<OpT>(D, jb.dst_sel) + jb.dst_off;
    if ((n & 3) == 0 && ((jb.dst_off & 3) == 0) && ((reinterpret_cast<uintptr_t>(jb.src) & 15) == 0)) {
      const float4* s4 = reinterpret_cast<const float4*>(jb.src);
      for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = s4[i];
        FV<4> f;
        f.v[0] = v.x; f.v[1] = v.y; f.v[2] = v.z; f.v[3] = v.w;
        stv_op<OpT, 4>(dst + 4 * i, f, D.ps_w[jb.dst_sel]);
      }
    } else {
      for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        st_op1<OpT>(dst + i, jb.src[i], D.ps_w[jb.dst_sel]);
    }
  }
}

// One CTA per 64-position tile; 4 consecutive x values per thread and step (16-byte loads).
// A grid of at most two tiles per SM (cfg4: ~148 tiles) runs 512 threads (8 loads of 16 B each in
// flight: ~64 KB per SM, what HBM latency x bandwidth asks for); larger grids keep 256 (several
// CTAs per SM already; 512 measured slower on cfg5's 511 tiles)
template <class OpT>
__global__ void k_pull(Dev D) {
  pdl_wait();
  if (D.hdr[0]) return;                          // invalid graphs: order[] is stale, touch nothing
  const int p0 = blockIdx.x * 64;
  __shared__ int s_r[64];
  if (threadIdx.x < 64) {
    const int p = p0 + threadIdx.x;
    int r = -1;
    if (p < D.V) {
      r = D.x_row[D.order[p]];
      if (r < -1 || r >= D.n_x) {                // out-of-range record: deferred CAVS_E_INVALID (cavs_sync),
        atomicOr(D.hdr + 3, ST_XROW);            // the vertex pulls nothing meanwhile
        r = -1;
      }
      D.xrow_pos[p] = r;
      if (r >= 0 && atomicExch(D.xseen + r, (int)D.xgen) == (int)D.xgen) D.hdr[5] = 1;   // a record pulled twice
    }
    s_r[threadIdx.x] = r;
    const unsigned has = __ballot_sync(0xffffffffu, r >= 0);   // warps 0-1: count this block's pulls
    if ((threadIdx.x & 31) == 0 && has) atomicAdd(D.hdr + 4, __popc(has));
  }
  const int any = __syncthreads_or(threadIdx.x < 64 && s_r[threadIdx.x] >= 0);
  if (threadIdx.x == 0) D.tile_x[blockIdx.x] = any;
  OpT* X = op<OpT>(D.Xp);
  const int d = D.d;
  if ((d & 3) == 0) {
    // 8 independent 16-byte loads in flight per thread (the copy is latency-bound otherwise)
    const int d4 = d >> 2, n = 64 * d4;
    for (int e0 = threadIdx.x; e0 < n; e0 += 8 * blockDim.x) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x, rr = e / d4, k = (e % d4) * 4;
        const int r = (e < n && p0 + rr < D.V) ? s_r[rr] : -1;
        v[u] = r >= 0 ? *reinterpret_cast<const float4*>(D.x + (size_t)r * d + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x, rr = e / d4, k = (e % d4) * 4;
        if (e >= n || p0 + rr >= D.V) continue;
        FV<4> f;
        f.v[0] = v[u].x; f.v[1] = v[u].y; f.v[2] = v[u].z; f.v[3] = v[u].w;
        stv_op<OpT, 4>(X + (size_t)(p0 + rr) * d + k, f, D.ps_xp);
      }
    }
  } else {
    for (int e = threadIdx.x; e < 64 * d; e += blockDim.x) {
      const int rr = e / d, k = e % d, p = p0 + rr;
      if (p >= D.V) break;
      const int r = s_r[rr];
      st_op1<OpT>(X + (size_t)p * d + k, r >= 0 ? D.x[(size_t)r * d + k] : 0.f, D.ps_xp);
    }
  }
}

template <class OpT>
__global__ void k_roots(Dev D, int n_roots, const int* roots) {
  pdl_wait();
  // PDL: the persistent backward's prologue (weights -> TMEM) may overlap this kernel (its
  // griddepcontrol.wait orders the reads of these dZ rows)
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (dev_skip(D)) return;
  if (n_roots < 0) n_roots = D.hdr[2];                      // sync-free mode: the device count
  const size_t n = (size_t)n_roots * D.h;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    root_bwd<OpT>(D, (int)(i % D.h), roots[i / D.h]);
  }
}

// db (P:L541-542 lazy batching of the bias gradient): db_g = sum over all vertices of dz_g.
// Logical columns L = (i, o, u, f) x h for Tree-LSTM (f summed over the N child slots: the
// shared U_f / b_f of Z6) or h for Tree-FC.  part[c][L] = sum over the rows of chunk c; CTA = 8
// warps x 256 logical columns, a lane owns 8 consecutive columns (16-byte loads per row in BF16
// mode), warp w takes rows w, w+8, ... of the chunk, the 8 warp partials are added in a fixed
// order.  The last CTA of a column block (arrival counter) sums the kDbChunks partials in chunk
// order and writes the packed db block of dparams (deterministic).
template <class OpT>
__global__ void __launch_bounds__(256) k_colsum(Dev D, float* part, int lcols) {
  pdl_wait();
  if (dev_skip(D)) return;
  __shared__ float red[8][256];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = D.h;
  const bool lstm = D.cell == CAVS_CELL_TREE_LSTM;
  const int cols = lstm ? (3 + D.N) * h : h;                 // physical dZ row width
  const int L0 = blockIdx.x * 256 + lane * 8;
  // blockIdx.y = (slot k, row chunk): the N child slots of the f block are summed by different
  // CTAs (balanced work); the other blocks' CTAs with k > 0 contribute zero partials
  const int kk = blockIdx.y / kDbChunks, cy = blockIdx.y % kDbChunks;
  const int chunk = cdiv(D.V, kDbChunks);
  const int r0 = cy * chunk, r1 = min(D.V, r0 + chunk);
  const OpT* dz = op<OpT>(D.dZ);
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (L0 + 8 <= lcols && (h & 7) == 0) {                     // 8 columns inside one gate
    const int gl = L0 / h, j = L0 - gl * h;
    const int nk = (lstm && gl == 3) ? D.N : 1;
    const int pc = (lstm && gl == 3) ? 3 * h + j : gl * h + j;
    for (int k = kk; k < min(nk, kk + 1); ++k) {
      const OpT* col = dz + pc + k * h;
      if constexpr (is_s3<OpT>::value) {                     // FP32 split mode: b0 + b1 + b2 per element
        for (int r = r0 + warp; r < r1; r += 8) {
          const OpT* rowp = col + (size_t)r * cols;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += ld_op1<OpT>(rowp + e, D.ps_dz);
        }
      } else if constexpr (sizeof(OpT) == 2) {
        int r = r0 + warp;
        for (; r + 56 < r1; r += 64) {                      // 8 rows in flight
          uint4 u[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) u[q] = *reinterpret_cast<const uint4*>(col + (size_t)(r + 8 * q) * cols);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(b2[e]); acc[2 * e] += f.x; acc[2 * e + 1] += f.y; }
          }
        }
        for (; r < r1; r += 8) {
          const uint4 u = *reinterpret_cast<const uint4*>(col + (size_t)r * cols);
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) { const float2 f = __bfloat1622float2(b2[e]); acc[2 * e] += f.x; acc[2 * e + 1] += f.y; }
        }
      } else {
        for (int r = r0 + warp; r < r1; r += 8) {
          const OpT* rowp = col + (size_t)r * cols;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += from_op(rowp[e]);
        }
      }
    }
  } else {
    for (int e = 0; e < 8 && L0 + e < lcols; ++e) {
      const int L = L0 + e, gl = L / h, j = L - gl * h;
      const int nk = (lstm && gl == 3) ? D.N : 1;
      const int pc = (lstm && gl == 3) ? 3 * h + j : gl * h + j;
      for (int k = kk; k < min(nk, kk + 1); ++k)
        for (int r = r0 + warp; r < r1; r += 8) acc[e] += ld_op1<OpT>(dz + (size_t)r * cols + pc + k * h, D.ps_dz);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[warp][lane * 8 + e] = acc[e];
  __syncthreads();
  const int L = blockIdx.x * 256 + threadIdx.x;
  if (L < lcols) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    part[(size_t)blockIdx.y * lcols + L] = v;
  }
  __threadfence();
  __syncthreads();
  int* cnt = D.tile_cnt + kLazyMaxTiles + blockIdx.x;
  if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1) == (int)gridDim.y - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (L < lcols) {
    float v = 0.f;
    for (int c0 = 0; c0 < (int)gridDim.y; c0 += 32) {       // 32 partials in flight, summed in chunk order
      float t[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) t[e] = c0 + e < (int)gridDim.y ? __ldcg(part + (size_t)(c0 + e) * lcols + L) : 0.f;
#pragma unroll
      for (int e = 0; e < 32; ++e) v += t[e];
    }
    const size_t H = h, Dd = D.d;
    if (lstm) {
      const int gl = L / h, j = L - gl * h;
      const int blk[4] = {0, 2, 3, 1};                       // internal (i, o, u, f) -> packed (i, f, o, u)
      D.dparams[4 * H * Dd + 4 * H * H + (size_t)blk[gl] * H + j] = v;
    } else {
      D.dparams[2 * H * H + H * Dd + L] = v;
    }
  }
  if (threadIdx.x == 0) *cnt = 0;                             // replayable
}

// Packing as segments: out[o0 + e] = sum_{s < S} sum_{q < nb} src[s * sstride + soff + q * qstride + e]
struct PackSeg { const float* src; size_t sstride, soff, qstride, o0; int S, nb, len; };
struct PackSegs { int n; PackSeg s[10]; };

__global__ void __launch_bounds__(256) k_pack(Dev D, PackSegs P) {
  const PackSeg& g = P.s[blockIdx.y];
  float* out = D.dparams + g.o0;
  // 4 consecutive outputs per thread and step, float4 loads when aligned; partials of a slot
  // are loaded together before they are added (fixed order: deterministic)
  const bool vec = ((g.len | g.sstride | g.soff | g.qstride | g.o0) & 3) == 0;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) * 4; e < g.len; e += gridDim.x * blockDim.x * 4) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < g.S; ++s)
      for (int q = 0; q < g.nb; ++q) {
        const float* src = g.src + s * g.sstride + g.soff + q * g.qstride + e;
        if (vec) {
          const float4 x = *reinterpret_cast<const float4*>(src);
          v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
        } else {
          v.x += src[0];
          if (e + 1 < g.len) v.y += src[1];
          if (e + 2 < g.len) v.z += src[2];
          if (e + 3 < g.len) v.w += src[3];
        }
      }
    if (vec) *reinterpret_cast<float4*>(out + e) = v;
    else {
      out[e] = v.x;
      if (e + 1 < g.len) out[e + 1] = v.y;
      if (e + 2 < g.len) out[e + 2] = v.z;
      if (e + 3 < g.len) out[e + 3] = v.w;
    }
  }
}

// ---- DAG inputs (D.dag): parent CSR by position ------------------------------------------
// count parents per child position, exclusive scan, fill, then sort every (short) list so the
// order of the pull-reduce is fixed: ascending parent-slot index q = parent_pos * N + k.
__global__ void k_dag_count(Dev D) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < D.V; p += gridDim.x * blockDim.x) {
    const int deg = D.deg[p];
    for (int k = 0; k < deg; ++k) atomicAdd(&D.pcur[D.child_pos[(size_t)p * D.N + k]], 1);
  }
}
__global__ void __launch_bounds__(1024) k_dag_scan(Dev D) {   // one CTA
  __shared__ int s_warp[32];
  int carry = 0;
  for (int b0 = 0; b0 < D.V; b0 += blockDim.x) {
    const int p = b0 + threadIdx.x;
    const int c = p < D.V ? D.pcur[p] : 0;
    int v = c;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(~0u, v, o); if (lane >= o) v += y; }
    if (lane == 31) s_warp[w] = v;
    __syncthreads();
    if (w == 0) {
      int y = lane < nw ? s_warp[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) { const int z = __shfl_up_sync(~0u, y, o); if (lane >= o) y += z; }
      s_warp[lane] = y;
    }
    __syncthreads();
    const int excl = carry + v - c + (w ? s_warp[w - 1] : 0);
    if (p < D.V) { D.pptr[p] = excl; D.pcur[p] = 0; }
    carry += s_warp[nw - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) D.pptr[D.V] = carry;
}
__global__ void k_dag_fill(Dev D) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < D.V; p += gridDim.x * blockDim.x) {
    const int deg = D.deg[p];
    for (int k = 0; k < deg; ++k) {
      const int c = D.child_pos[(size_t)p * D.N + k];
      D.pent[D.pptr[c] + atomicAdd(&D.pcur[c], 1)] = p * D.N + k;
    }
  }
}
__global__ void k_dag_sort(Dev D) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < D.V; p += gridDim.x * blockDim.x) {
    const int a = D.pptr[p], b = D.pptr[p + 1];
    for (int i = a + 1; i < b; ++i) {              // insertion sort: lists are short
      const int x = D.pent[i];
      int j = i - 1;
      while (j >= a && D.pent[j] > x) { D.pent[j + 1] = D.pent[j]; --j; }
      D.pent[j + 1] = x;
    }
    D.pcur[p] = 0;                                 // cursors zero for the next batch
  }
}

// Forward gather of task [lo, hi): slot k of parent p <- the child's pushed h (operand dtype) and c.
template <class OpT>
__global__ void k_dag_gather(Dev D, int lo, int hi) {
  const int h = D.h, N = D.N;
  const size_t n = (size_t)(hi - lo) * N * h;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % h);
    const int k = (int)((i / h) % N);
    const int p = lo + (int)(i / ((size_t)N * h));
    if (k >= D.deg[p]) continue;                   // missing slots stay zero (k_build_maps, Z1)
    const int c = D.child_pos[(size_t)p * N + k];
    const size_t at = ((size_t)p * N + k) * h + j;
    st_op1<OpT>(op<OpT>(D.Hk) + at, D.h_out[(size_t)D.order[c] * h + j], D.ps_hk);
    if (D.Ck) D.Ck[at] = D.cst[(size_t)c * h + j];
  }
}

// Backward pull-reduce + dF of task [lo, hi) (cells.cuh dag_df).
template <class OpT>
__global__ void k_dag_df(Dev D, int lo, int hi) {
  const size_t n = (size_t)(hi - lo) * D.h;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dag_df<OpT>(D, (int)(i % D.h), lo + (int)(i / D.h));
}

// Unfused ablation (CAVS_UNFUSED=1): the cell's elementwise part as its own kernel,
// reading the level GEMM's raw accumulators (one thread per (vertex, unit)).
template <int E, class OpT>
__global__ void k_unfused(Dev D, int lo, int hi) {
  const int h = D.h, nacc = D.rawld / h;
  const size_t n = (size_t)(hi - lo) * h;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % h), p = lo + (int)(i / h);
    VMeta m;
    load_meta(D, p, epi_needs_children<E>(), m);
    FV<1> acc[3 + kMaxN];
#pragma unroll
    for (int e = 0; e < 3 + kMaxN; ++e) acc[e].v[0] = e < nacc ? D.raw[(size_t)p * D.rawld + (size_t)e * h + j] : 0.f;
    const UnitC<1> uc = epi_uses_bias<E>() ? load_unit<1>(D, j, epi_is_lstm<E>()) : UnitC<1>{};
    typename EpiK<E>::template In<1, kMaxN> in;
    EpiK<E>::template load<1, kMaxN>(D, j, m, in);
    EpiK<E>::template store<OpT, 1, kMaxN>(D, j, m, acc, in, uc);
  }
}

template <class OpT>
static void unfused_t(const Dev& D, int epi, int lo, int hi, int g, cudaStream_t s) {
  switch (epi) {
    case EPI_LSTM_FWD: k_unfused<EPI_LSTM_FWD, OpT><<<g, 256, 0, s>>>(D, lo, hi); break;
    case EPI_LSTM_BWD: k_unfused<EPI_LSTM_BWD, OpT><<<g, 256, 0, s>>>(D, lo, hi); break;
    case EPI_FC_FWD: k_unfused<EPI_FC_FWD, OpT><<<g, 256, 0, s>>>(D, lo, hi); break;
    case EPI_FC_BWD: k_unfused<EPI_FC_BWD, OpT><<<g, 256, 0, s>>>(D, lo, hi); break;
    case EPI_LSTM_BWD_DAG: k_unfused<EPI_LSTM_BWD_DAG, OpT><<<g, 256, 0, s>>>(D, lo, hi); break;
    case EPI_FC_BWD_DAG: k_unfused<EPI_FC_BWD_DAG, OpT><<<g, 256, 0, s>>>(D, lo, hi); break;
    default: break;
  }
}

// dst[rows[i]] = src[i] for n rows of w floats (the push cotangents of the loss vertices)
__global__ void k_scatter_rows(float* dst, const float* src, const int* rows, int n, int w) {
  const size_t tot = (size_t)n * w;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x)
    dst[(size_t)rows[i / w] * w + i % w] = src[i];
}

// dx must be zeroed unless every record is pulled exactly once (then every row gets one store)
__global__ void k_dx_zero(Dev D) {
  pdl_wait();
  if (!D.hdr[5] && D.hdr[4] == D.n_x) return;
  const size_t n = (size_t)D.n_x * D.d;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(D.dx) & 15) == 0) {
    float4* d4 = reinterpret_cast<float4*>(D.dx);
    for (size_t i = tid; i < n / 4; i += stride) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    for (size_t i = tid; i < n; i += stride) D.dx[i] = 0.f;
  }
}

static int grid_for(size_t n, int block) { return (int)std::min<size_t>((n + block - 1) / block, 148 * 16); }

void launch_prep(const Dev& D, cudaStream_t s) {
  const size_t h = D.h, d = D.d;
  const int N = D.N;
  PrepJobs J{};
  auto add = [&](const float* src, int rows, int cols, int spitch, int sel, size_t off, int dpitch, int tr) {
    J.j[J.n++] = PrepJob{src, rows, cols, spitch, sel, off, dpitch, tr};
  };
  const float* t = D.params;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    const int G = 3 + N;
    const float* W = t;                       // [4h x d] blocks (i, f, o, u)
    const float* Uiou = t + 4 * h * d;        // [3h x h] (i, o, u)
    const float* Uf = Uiou + 3 * h * h;       // [h x h]
    const float* b = Uf + h * h;              // [4h] (i, f, o, u)
    const int blkW[4] = {0, 2, 3, 1};         // internal gate (i, o, u, f) -> packed block
    add(Uiou, 1, (int)(4 * h * h), 0, 0, 0, 0, 0);                                   // U4 = [U_iou; U_f]
    for (int g = 0; g < 4; ++g) add(W + blkW[g] * h * d, 1, (int)(h * d), 0, 1, g * h * d, 0, 0);   // W4
    add(Uiou, (int)(3 * h), (int)h, (int)h, 2, 0, (int)(3 * h), 1);                  // UTiou = U_iou^T
    add(Uf, (int)h, (int)h, (int)h, 3, 0, (int)h, 1);                                // UTf = U_f^T
    for (int g = 0; g < G; ++g)                                                      // WT[:, g h] = W_g^T
      add(W + blkW[g < 3 ? g : 3] * h * d, (int)h, (int)d, (int)d, 4, g * h, G * (int)h, 1);
    for (int g = 0; g < 4; ++g) add(b + blkW[g] * h, 1, (int)h, 0, 5, g * h, 0, 0);
  } else {
    const float* Wc = t;                      // [h x 2h]
    const float* Wx = t + 2 * h * h;          // [h x d]
    const float* b = Wx + h * d;
    add(Wc, 1, (int)(2 * h * h), 0, 0, 0, 0, 0);
    add(Wx, 1, (int)(h * d), 0, 1, 0, 0, 0);
    add(Wc, (int)h, (int)(2 * h), (int)(2 * h), 2, 0, (int)h, 1);                    // WcT = W_c^T [2h x h]
    add(Wx, (int)h, (int)d, (int)d, 4, 0, (int)h, 1);                                // WxT = W_x^T [d x h]
    add(b, 1, (int)h, 0, 5, 0, 0, 0);
  }
  dim3 grid(148, J.n);
  if (D.prec == CAVS_BF16) launch_pdl(k_prep<__nv_bfloat16>, grid, dim3(256), 0, s, D, J);
  else if (D.split) launch_pdl(k_prep<S3>, grid, dim3(256), 0, s, D, J);
  else launch_pdl(k_prep<float>, grid, dim3(256), 0, s, D, J);
}

void launch_pull(const Dev& D, cudaStream_t s) {
  static int n_sm[kMaxDev] = {};
  const int dv = cur_device();
  if (!n_sm[dv]) cudaDeviceGetAttribute(&n_sm[dv], cudaDevAttrMultiProcessorCount, dv);
  const int nt = cdiv(D.V, 64) <= 2 * n_sm[dv] ? 512 : 256;
  if (D.prec == CAVS_BF16) launch_pdl(k_pull<__nv_bfloat16>, dim3(cdiv(D.V, 64)), dim3(nt), 0, s, D);
  else if (D.split) launch_pdl(k_pull<S3>, dim3(cdiv(D.V, 64)), dim3(nt), 0, s, D);
  else launch_pdl(k_pull<float>, dim3(cdiv(D.V, 64)), dim3(nt), 0, s, D);
}

void launch_roots(const Dev& D, int n_roots, const int* roots, cudaStream_t s) {
  const size_t n = (size_t)(n_roots < 0 ? D.V : n_roots) * D.h;   // < 0: device count, grid for V
  if (D.prec == CAVS_BF16) launch_pdl(k_roots<__nv_bfloat16>, dim3(grid_for(n, 256)), dim3(256), 0, s, D, n_roots, roots);
  else if (D.split) launch_pdl(k_roots<S3>, dim3(grid_for(n, 256)), dim3(256), 0, s, D, n_roots, roots);
  else launch_pdl(k_roots<float>, dim3(grid_for(n, 256)), dim3(256), 0, s, D, n_roots, roots);
}

void launch_colsum(const Dev& D, float* part, cudaStream_t s) {
  const int lcols = (D.cell == CAVS_CELL_TREE_LSTM ? 4 : 1) * D.h;
  dim3 grid(cdiv(lcols, 256), kDbChunks * (D.cell == CAVS_CELL_TREE_LSTM ? D.N : 1));   // (slot, row chunk)
  if (D.prec == CAVS_BF16) launch_pdl(k_colsum<__nv_bfloat16>, grid, dim3(256), 0, s, D, part, lcols);
  else if (D.split) launch_pdl(k_colsum<S3>, grid, dim3(256), 0, s, D, part, lcols);
  else launch_pdl(k_colsum<float>, grid, dim3(256), 0, s, D, part, lcols);
}

void launch_pack(const Dev& D, const int* split, cudaStream_t s) {
  const LazyLayout Z = lazy_layout(D);
  const size_t h = D.h, d = D.d;
  const int N = D.N;
  PackSegs P{};
  const float* u4 = D.lazy + Z.u4;
  const float* uf = D.lazy + Z.uf;
  const float* w = D.lazy + Z.w;
  int maxlen = 0;
  auto add = [&](const float* src, size_t sstride, size_t soff, size_t qstride, size_t o0, int S, int nb, size_t len) {
    P.s[P.n++] = PackSeg{src, sstride, soff, qstride, o0, S, nb, (int)len};
    maxlen = std::max(maxlen, (int)len);
  };
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    const int G = 3 + N;
    const int intern[4] = {0, 3, 1, 2};      // packed (i, f, o, u) -> internal row block (f: 3..3+N-1)
    const size_t nW = 4 * h * d, nU = 3 * h * h, nUf = h * h;
    for (int pg = 0; pg < 4; ++pg)           // W blocks: sum over split slots (and the N f-blocks)
      add(w, Z.sw, intern[pg] * h * d, h * d, pg * h * d, split[2], pg == 1 ? N : 1, h * d);
    add(u4, Z.su4, 0, 0, nW, split[0], 1, nU);
    add(uf, Z.suf, 0, 0, nW + nU, split[1], 1, nUf);
  } else {
    add(u4, Z.su4, 0, 0, 0, split[0], 1, 2 * h * h);
    add(w, Z.sw, 0, 0, 2 * h * h, split[2], 1, h * d);
  }
  dim3 grid(std::min(148, cdiv(maxlen, 256 * 4)), P.n);
  k_pack<<<grid, 256, 0, s>>>(D, P);
}

void launch_dag_parents(const Dev& D, cudaStream_t s) {
  const int g = grid_for(D.V, 256);
  k_dag_count<<<g, 256, 0, s>>>(D);
  k_dag_scan<<<1, 1024, 0, s>>>(D);
  k_dag_fill<<<g, 256, 0, s>>>(D);
  k_dag_sort<<<g, 256, 0, s>>>(D);
}

void launch_dag_gather(const Dev& D, int lo, int hi, cudaStream_t s) {
  if (hi <= lo) return;
  const size_t n = (size_t)(hi - lo) * D.N * D.h;
  if (D.prec == CAVS_BF16) k_dag_gather<__nv_bfloat16><<<grid_for(n, 256), 256, 0, s>>>(D, lo, hi);
  else if (D.split) k_dag_gather<S3><<<grid_for(n, 256), 256, 0, s>>>(D, lo, hi);
  else k_dag_gather<float><<<grid_for(n, 256), 256, 0, s>>>(D, lo, hi);
}

void launch_dag_df(const Dev& D, int lo, int hi, cudaStream_t s) {
  if (hi <= lo) return;
  const size_t n = (size_t)(hi - lo) * D.h;
  if (D.prec == CAVS_BF16) k_dag_df<__nv_bfloat16><<<grid_for(n, 256), 256, 0, s>>>(D, lo, hi);
  else if (D.split) k_dag_df<S3><<<grid_for(n, 256), 256, 0, s>>>(D, lo, hi);
  else k_dag_df<float><<<grid_for(n, 256), 256, 0, s>>>(D, lo, hi);
}

void launch_unfused(const Dev& D, int epi, int lo, int hi, cudaStream_t s) {
  if (hi <= lo) return;
  const int g = grid_for((size_t)(hi - lo) * D.h, 256);
  if (D.prec == CAVS_BF16) unfused_t<__nv_bfloat16>(D, epi, lo, hi, g, s);
  else unfused_t<float>(D, epi, lo, hi, g, s);
}

void launch_scatter_rows(float* dst, const float* src, const int* rows, int n, int w, cudaStream_t s) {
  if (n <= 0) return;
  k_scatter_rows<<<grid_for((size_t)n * w, 256), 256, 0, s>>>(dst, src, rows, n, w);
}

void launch_dx_zero(const Dev& D, cudaStream_t s) {
  // usually an early exit (every record pulled once): a small grid keeps the launch cheap
  launch_pdl(k_dx_zero, dim3(std::min(grid_for((size_t)D.n_x * D.d / 4 + 1, 256), 2 * 148)), dim3(256), 0, s, D);
}

}  // namespace cavs
