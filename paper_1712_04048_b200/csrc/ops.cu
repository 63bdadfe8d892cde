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

template <class OpT>
__global__ void k_prep(Dev D) {
  const int h = D.h, d = D.d, N = D.N;
  const float* t = D.params;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    // packed: W[4h x d] rows (i,f,o,u) | U_iou[3h x h] (i,o,u) | U_f[h x h] | b[4h] (i,f,o,u)
    const float* W = t;
    const float* Uiou = t + (size_t)4 * h * d;
    const float* Uf = Uiou + (size_t)3 * h * h;
    const float* b = Uf + (size_t)h * h;
    const int blkW[4] = {0, 2, 3, 1};           // internal gate (i,o,u,f) -> packed W/b block
    OpT* U4 = op<OpT>(D.Wa); OpT* W4 = op<OpT>(D.Wb); OpT* UTiou = op<OpT>(D.Wc);
    OpT* UTf = op<OpT>(D.Wd); OpT* WT = op<OpT>(D.We);
    const int G = 3 + N;
    for (size_t i = i0; i < (size_t)4 * h * h; i += stride) {      // U4[g*h+m][k]
      const int r = (int)(i / h), k = (int)(i % h), g = r / h, m = r % h;
      U4[i] = to_op<OpT>(g < 3 ? Uiou[(size_t)(g * h + m) * h + k] : Uf[(size_t)m * h + k]);
    }
    for (size_t i = i0; i < (size_t)4 * h * d; i += stride) {      // W4[g*h+m][k]
      const int r = (int)(i / d), k = (int)(i % d), g = r / h, m = r % h;
      W4[i] = to_op<OpT>(W[(size_t)(blkW[g] * h + m) * d + k]);
    }
    for (size_t i = i0; i < (size_t)3 * h * h; i += stride) {      // UTiou[j][g*h+m] = U_g[m][j]
      const int j = (int)(i / (3 * h)), c = (int)(i % (3 * h));
      UTiou[i] = to_op<OpT>(Uiou[(size_t)c * h + j]);
    }
    for (size_t i = i0; i < (size_t)h * h; i += stride) {          // UTf[j][m] = U_f[m][j]
      const int j = (int)(i / h), m = (int)(i % h);
      UTf[i] = to_op<OpT>(Uf[(size_t)m * h + j]);
    }
    for (size_t i = i0; i < (size_t)d * G * h; i += stride) {      // WT[j][g*h+m] = W_g[m][j]
      const int j = (int)(i / (G * h)), c = (int)(i % (G * h)), g = c / h, m = c % h;
      WT[i] = to_op<OpT>(W[(size_t)(blkW[g < 3 ? g : 3] * h + m) * d + j]);
    }
    for (size_t i = i0; i < (size_t)4 * h; i += stride) {
      const int g = (int)(i / h), m = (int)(i % h);
      D.bias[i] = b[blkW[g] * h + m];
    }
  } else {
    // packed: W_c[h x 2h] | W_x[h x d] | b[h]
    const float* Wcp = t;
    const float* Wx = t + (size_t)2 * h * h;
    const float* b = Wx + (size_t)h * d;
    OpT* Wc = op<OpT>(D.Wa); OpT* Wxo = op<OpT>(D.Wb); OpT* WcT = op<OpT>(D.Wc); OpT* WxT = op<OpT>(D.We);
    for (size_t i = i0; i < (size_t)2 * h * h; i += stride) {
      Wc[i] = to_op<OpT>(Wcp[i]);
      const int r = (int)(i / h), m = (int)(i % h);              // WcT[k*h+j][m] = Wc[m][k*h+j]
      WcT[i] = to_op<OpT>(Wcp[(size_t)m * 2 * h + r]);
    }
    for (size_t i = i0; i < (size_t)h * d; i += stride) {
      Wxo[i] = to_op<OpT>(Wx[i]);
      const int j = (int)(i / h), m = (int)(i % h);              // WxT[j][m] = Wx[m][j]
      WxT[i] = to_op<OpT>(Wx[(size_t)m * d + j]);
    }
    for (size_t i = i0; i < (size_t)h; i += stride) D.bias[i] = b[i];
  }
}

// One CTA per 64-position tile; 4 consecutive x values per thread and step (16-byte loads).
template <class OpT>
__global__ void k_pull(Dev D) {
  const int p0 = blockIdx.x * 64;
  __shared__ int s_r[64];
  if (threadIdx.x < 64) {
    const int p = p0 + threadIdx.x;
    int r = -1;
    if (p < D.V) {
      r = D.x_row[D.order[p]];
      if (r >= D.n_x) r = -1;                    // out-of-range record: treated as absent
      D.xrow_pos[p] = r;
    }
    s_r[threadIdx.x] = r;
  }
  const int any = __syncthreads_or(threadIdx.x < 64 && s_r[threadIdx.x] >= 0);
  if (threadIdx.x == 0) D.tile_x[blockIdx.x] = any;
  OpT* X = op<OpT>(D.Xp);
  const int d = D.d;
  if ((d & 3) == 0) {
    const int d4 = d >> 2;
    for (int e = threadIdx.x; e < 64 * d4; e += blockDim.x) {
      const int rr = e / d4, k = (e % d4) * 4, p = p0 + rr;
      if (p >= D.V) break;
      const int r = s_r[rr];
      const float4 v = r >= 0 ? *reinterpret_cast<const float4*>(D.x + (size_t)r * d + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      OpT* o = X + (size_t)p * d + k;
      o[0] = to_op<OpT>(v.x); o[1] = to_op<OpT>(v.y); o[2] = to_op<OpT>(v.z); o[3] = to_op<OpT>(v.w);
    }
  } else {
    for (int e = threadIdx.x; e < 64 * d; e += blockDim.x) {
      const int rr = e / d, k = e % d, p = p0 + rr;
      if (p >= D.V) break;
      const int r = s_r[rr];
      X[(size_t)p * d + k] = to_op<OpT>(r >= 0 ? D.x[(size_t)r * d + k] : 0.f);
    }
  }
}

template <class OpT>
__global__ void k_roots(Dev D, int n_roots, const int* roots) {
  const size_t n = (size_t)n_roots * D.h;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    root_bwd<OpT>(D, (int)(i % D.h), roots[i / D.h]);
  }
}

// part[c][col] = sum over rows of chunk c of dZ[row][col]
template <class OpT>
__global__ void k_colsum(Dev D, float* part, int cols) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= cols) return;
  const int chunk = cdiv(D.V, gridDim.y);
  const int r0 = blockIdx.y * chunk, r1 = min(D.V, r0 + chunk);
  const OpT* dz = op<OpT>(D.dZ);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int r = r0;
  for (; r + 3 < r1; r += 4) {
    s0 += from_op(dz[(size_t)r * cols + col]);
    s1 += from_op(dz[(size_t)(r + 1) * cols + col]);
    s2 += from_op(dz[(size_t)(r + 2) * cols + col]);
    s3 += from_op(dz[(size_t)(r + 3) * cols + col]);
  }
  for (; r < r1; ++r) s0 += from_op(dz[(size_t)r * cols + col]);
  part[(size_t)blockIdx.y * cols + col] = (s0 + s1) + (s2 + s3);
}

__global__ void k_pack(Dev D, LazyLayout Z, int Su4, int Suf, int Sw, const float* dbp) {
  const int h = D.h, d = D.d, N = D.N;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  float* out = D.dparams;
  const float* u4 = D.lazy + Z.u4;
  const float* uf = D.lazy + Z.uf;
  const float* w = D.lazy + Z.w;
  if (D.cell == CAVS_CELL_TREE_LSTM) {
    const int G = 3 + N;
    const size_t nW = (size_t)4 * h * d, nU = (size_t)3 * h * h, nUf = (size_t)h * h;
    const int intern[4] = {0, 3, 1, 2};         // packed (i,f,o,u) -> internal row block (f: 3..3+N-1)
    for (size_t i = i0; i < nW + nU + nUf + 4 * h; i += stride) {
      float v = 0.f;
      if (i < nW) {
        const int pg = (int)(i / ((size_t)h * d)); const size_t rest = i % ((size_t)h * d);
        const int nb = pg == 1 ? N : 1;
        for (int s = 0; s < Sw; ++s)
          for (int q = 0; q < nb; ++q) v += w[s * Z.sw + (size_t)(intern[pg] + q) * h * d + rest];
      } else if (i < nW + nU) {
        const size_t r = i - nW;
        for (int s = 0; s < Su4; ++s) v += u4[s * Z.su4 + r];
      } else if (i < nW + nU + nUf) {
        const size_t r = i - nW - nU;
        for (int s = 0; s < Suf; ++s) v += uf[s * Z.suf + r];
      } else {
        const size_t r = i - nW - nU - nUf;
        const int pg = (int)(r / h), m = (int)(r % h);
        const int nb = pg == 1 ? N : 1;
        for (int c = 0; c < kDbChunks; ++c)
          for (int q = 0; q < nb; ++q) v += dbp[(size_t)c * G * h + (size_t)(intern[pg] + q) * h + m];
      }
      out[i] = v;
    }
  } else {
    const size_t swc = Z.su4, swx = Z.sw;
    for (size_t i = i0; i < swc + swx + h; i += stride) {
      float v = 0.f;
      if (i < swc) { for (int s = 0; s < Su4; ++s) v += u4[s * swc + i]; }
      else if (i < swc + swx) { for (int s = 0; s < Sw; ++s) v += w[s * swx + (i - swc)]; }
      else { for (int c = 0; c < kDbChunks; ++c) v += dbp[(size_t)c * h + (i - swc - swx)]; }
      out[i] = v;
    }
  }
}

static int grid_for(size_t n, int block) { return (int)std::min<size_t>((n + block - 1) / block, 148 * 16); }

void launch_prep(const Dev& D, cudaStream_t s) {
  const size_t n = (size_t)4 * D.h * std::max(D.h, D.d) + (size_t)D.d * (3 + D.N) * D.h;
  if (D.prec == CAVS_BF16) k_prep<__nv_bfloat16><<<grid_for(n, 256), 256, 0, s>>>(D);
  else k_prep<float><<<grid_for(n, 256), 256, 0, s>>>(D);
}

void launch_pull(const Dev& D, cudaStream_t s) {
  if (D.prec == CAVS_BF16) k_pull<__nv_bfloat16><<<cdiv(D.V, 64), 256, 0, s>>>(D);
  else k_pull<float><<<cdiv(D.V, 64), 256, 0, s>>>(D);
}

void launch_roots(const Dev& D, int n_roots, const int* roots, cudaStream_t s) {
  const size_t n = (size_t)n_roots * D.h;
  if (D.prec == CAVS_BF16) k_roots<__nv_bfloat16><<<grid_for(n, 256), 256, 0, s>>>(D, n_roots, roots);
  else k_roots<float><<<grid_for(n, 256), 256, 0, s>>>(D, n_roots, roots);
}

void launch_colsum(const Dev& D, float* part, cudaStream_t s) {
  const int cols = (D.cell == CAVS_CELL_TREE_LSTM ? 3 + D.N : 1) * D.h;
  dim3 grid(cdiv(cols, 128), kDbChunks);   // 32 deterministic row chunks
  if (D.prec == CAVS_BF16) k_colsum<__nv_bfloat16><<<grid, 128, 0, s>>>(D, part, cols);
  else k_colsum<float><<<grid, 128, 0, s>>>(D, part, cols);
}

void launch_pack(const Dev& D, const int* split, const float* db_part, cudaStream_t s) {
  const size_t n = (size_t)4 * D.h * D.d + (size_t)4 * D.h * D.h + 4 * D.h;
  k_pack<<<grid_for(n, 256), 256, 0, s>>>(D, lazy_layout(D), split[0], split[1], split[2], db_part);
}

}  // namespace cavs
