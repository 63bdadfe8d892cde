// tools/mma_rate.cu — microbenchmark: cycles per tcgen05.mma (kind::f16, M = 128, K = 16) vs N,
// with A from shared memory (SS) or from TMEM (TS), B from shared memory; one CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1712_04048_b200/csrc tools/mma_rate.cu -o tools/mma_rate
#include <cuda_runtime.h>
#include <cstdio>

#include "ptx.cuh"

using namespace cavs;

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return ((uint64_t)((1024u >> 4) | (1u << 14) | (2u << 29)) << 32) | (((saddr >> 4) & 0x3FFF) | (1u << 16));
}

template <int N, bool TS>
__global__ void k_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  // A: 128 x 64 bf16 tile (16 KB) at smem, B: N x 64 (N*128 B) after it; contents irrelevant
  const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
  constexpr uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    if (TS && ptx::elect_one()) {
      for (int kk = 0; kk < 4; ++kk) ptx::tmem_cp_128x256b(tmem + 256 + kk * 8, desc(a + kk * 32));
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    if (TS) { ptx::mbar_wait(&bar, 0); ptx::tc_fence_after(); }
    const uint32_t ph = TS ? 1 : 0;
    if (ptx::elect_one()) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if constexpr (TS) ptx::mma_bf16_ts(tmem, tmem + 256 + kk * 8, desc(b + kk * 32), idesc, it | kk ? 1u : 0u);
          else ptx::mma_bf16(tmem, desc(a + kk * 32), desc(b + kk * 32), idesc, it | kk ? 1u : 0u);
        }
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, ph);
    if (threadIdx.x == 0) { t1 = clock64(); out[blockIdx.x] = t1 - t0; }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

// k_rows-like issue (r02): SS M = 128 x N x 16 MMAs in k-blocks of 4, a tcgen05.commit to one of S
// rotating stage barriers after every `every` k-blocks (0: none), nothing waiting on them; is the
// commit itself a bubble in the tensor pipe?
template <int N>
__global__ void k_commit(int iters, int every, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, st[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&st[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
  constexpr uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
  if (warp == 0) {
    unsigned long long t0 = 0;
    if (ptx::elect_one()) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_bf16(tmem, desc(a + kk * 32), desc(b + kk * 32), idesc, it | kk ? 1u : 0u);
        if (every && (it + 1) % every == 0) ptx::mma_commit(&st[it & 3]);
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int N>
void run_commit(int every) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k_commit<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 512;
  k_commit<N><<<1, 128, smem>>>(iters, every, d);
  k_commit<N><<<1, 128, smem>>>(iters, every, d);
  cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("SS N=%3d commit every %d k-blocks: %6.1f cycles/MMA (floor %d)  err=%s\n", N, every, (double)h / (iters * 4),
         128 * N / 256, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

// persist-like issue: per tile 2 segments x 8 k-blocks x 4 MMAs (TS, N = 16), A walking 256 TMEM
// columns, B walking a 32 KB box (16 k-blocks of 16 rows), 2 accumulators; one commit per tile.
template <int N>
__global__ void k_tile_issue(int iters, unsigned long long* out, int wait_each, int noise) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ int slot2;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); slot2 = 0; }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t b = ptx::smem_u32(smem);
  constexpr uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
  unsigned long long t0 = 0;
  if (noise >= 3) {   // realistic operands: random bf16 in B (smem) and in A (TMEM columns 0..255)
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 16 * N * 32; i += blockDim.x) {
      uint32_t x = (uint32_t)i * 2654435761u + 12345u; x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      w[i] = (x & 0x3fff3fffu) | 0x3c003c00u;   // bf16 pairs in [1, 2)-ish with random mantissas
    }
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0 && ptx::elect_one()) {
      for (int c = 0; c < 32; ++c) ptx::tmem_cp_128x256b(tmem + c * 8, desc(b + (c % 16) * 32 * 4));
      ptx::mma_commit(&bar);
    }
    if (warp == 0) { __syncwarp(); ptx::mbar_wait(&bar, 0); ptx::tc_fence_after(); }
    __syncthreads();
  }
  if (warp == 0) {
    uint32_t ph = noise >= 3 ? 1 : 0;
    if (ptx::elect_one()) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        for (int g = 0; g < 16; ++g) {
          const uint32_t d = tmem + 256 + (g >> 3) * N;
          const uint32_t at = (uint32_t)(g & 7) * 32u;
          const uint32_t bl = b + (uint32_t)g * N * 128;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_bf16_ts(d, tmem + at + kk * 8, desc(bl + kk * 32), idesc, (g & 7) | kk ? 1u : 0u);
        }
        if (wait_each) { ptx::mma_commit(&bar); ptx::mbar_wait(&bar, ph); ph ^= 1; }
      }
      if (!wait_each) { ptx::mma_commit(&bar); ptx::mbar_wait(&bar, 0); }
      out[blockIdx.x] = clock64() - t0;
      *(volatile int*)&slot2 = 1;
    }
    __syncwarp();
  } else if (noise == 1) {                           // other warps spin on a shared-memory flag
    while (*(volatile int*)&slot2 == 0) { }
  } else if (noise == 2) {                           // other warps read TMEM (epilogue-like)
    const uint32_t q = (uint32_t)((warp & 3) * 32) << 16;
    while (*(volatile int*)&slot2 == 0) { uint32_t r[4]; asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tmem + q + 400)); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int N>
void run_tile(int wait_each, int noise = 0) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 16 * N * 128 + 1024;
  cudaFuncSetAttribute(k_tile_issue<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 64;
  k_tile_issue<N><<<1, noise ? 384 : 128, smem>>>(iters, d, wait_each, noise);
  k_tile_issue<N><<<1, noise ? 384 : 128, smem>>>(iters, d, wait_each, noise);
  cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("tile-issue N=%3d wait_each=%d noise=%d : %6.1f cycles/MMA (64 MMAs per tile)  err=%s\n", N, wait_each, noise, (double)h / (iters * 64),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

template <int N, bool TS>
void run(int grid) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 256;
  k_rate<N, TS><<<grid, 128, smem>>>(iters, d);
  k_rate<N, TS><<<grid, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per = (double)mx / (iters * 4);
  printf("%s N=%3d grid=%3d : %6.1f cycles/MMA  (%5.0f MAC/cycle/SM, %.0f%% of 4096)  err=%s\n", TS ? "TS" : "SS", N, grid,
         per, 128.0 * N * 16 / per, 100.0 * 128.0 * N * 16 / per / 4096, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'c') {       // ./mma_rate commit
    for (int e : {0, 1, 2, 4}) { run_commit<256>(e); run_commit<128>(e); run_commit<64>(e); }
    return 0;
  }
  for (int w : {0, 1}) { run_tile<16>(w); run_tile<32>(w); run_tile<64>(w); }
  for (int nz : {1, 2, 3}) { run_tile<16>(1, nz); run_tile<32>(1, nz); }
  return 0;
  for (int grid : {1, 148}) {
    run<16, false>(grid); run<32, false>(grid); run<64, false>(grid); run<128, false>(grid); run<256, false>(grid);
    run<16, true>(grid); run<32, true>(grid); run<64, true>(grid); run<128, true>(grid); run<256, true>(grid);
  }
  return 0;
}
