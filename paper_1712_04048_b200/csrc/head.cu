// head.cu — the external data path of Fig. 3 that turns the Fixed/Var-LSTM configs into language
// models: the next-word softmax head of PAPER.md §5 ("predicts the next
// word"), which lives OUTSIDE (F, G) (reading Z9) and is wired to F by push (h_out) and
// push's adjoint (dh_out).  The head's two contractions (logits = H W^T + b, dH = dlogits W) are
// plain GEMMs; this file is the fused softmax / cross-entropy / gradient pass over the logits.
//
//   loss_m    = logsumexp_c(logits[m, :]) - logits[m, target_m]      (rows with target_m < 0: 0)
//   dlogits_m = scale * (softmax(logits[m, :]) - onehot(target_m))   (may overwrite logits)
//
// One CTA per row: pass 1 reads the row once for its maximum and the sum of exp(l - max) in one
// online sweep (a running max rescales the running sum), pass 2 writes the gradient.  HBM bound:
// 2 reads + 1 write of M x vocab fp32.
#include <cfloat>

#include "kernels.h"

namespace cavs {

constexpr int kXentThreads = 512;

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mx = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * expf(m - mx)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mx));
  m = mx;
}

__global__ void __launch_bounds__(kXentThreads) k_softmax_xent(const float* logits, int vocab, const int* target,
                                                              float* loss, float* dlogits, float scale) {
  const int row = blockIdx.x;
  const float* l = logits + (size_t)row * vocab;
  const int tgt = target[row];
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x; c < vocab; c += blockDim.x) {
    const float x = l[c];
    if (x > m) { s = s * expf(m - x) + 1.f; m = x; }
    else s += expf(x - m);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(~0u, m, o), s2 = __shfl_xor_sync(~0u, s, o);
    online_merge(m, s, m2, s2);
  }
  __shared__ float sm[32], ss[32];
  __shared__ float s_lse;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sm[w] = m; ss[w] = s; }
  __syncthreads();
  if (w == 0) {
    m = lane < (int)(blockDim.x >> 5) ? sm[lane] : -INFINITY;
    s = lane < (int)(blockDim.x >> 5) ? ss[lane] : 0.f;
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(~0u, m, o), s2 = __shfl_xor_sync(~0u, s, o);
      online_merge(m, s, m2, s2);
    }
    if (lane == 0) {
      s_lse = m + logf(s);
      if (loss) loss[row] = tgt >= 0 ? s_lse - l[tgt] : 0.f;
    }
  }
  __syncthreads();
  const float lse = s_lse;
  float* d = dlogits + (size_t)row * vocab;
  for (int c = threadIdx.x; c < vocab; c += blockDim.x) {
    const float p = tgt >= 0 ? expf(l[c] - lse) : 0.f;
    d[c] = scale * (c == tgt ? p - 1.f : p);
  }
}

}  // namespace cavs

extern "C" __attribute__((visibility("default")))
cavs_status cavs_softmax_xent(const float* logits, int32_t M, int32_t vocab, const int32_t* target, float* loss,
                              float* dlogits, float scale, void* stream) {
  if (M < 0 || vocab < 1 || (M > 0 && (!logits || !target || !dlogits))) return CAVS_E_INVALID;
  if (M == 0) return CAVS_OK;
  cavs::k_softmax_xent<<<M, cavs::kXentThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(logits, vocab, target,
                                                                                            loss, dlogits, scale);
  return cudaGetLastError() == cudaSuccess ? CAVS_OK : CAVS_E_CUDA;
}
