// tools/tma_tile.cu — microbenchmark: latency of loading one B tile of the persistent level
// kernel (NT rows x 8 k-blocks of a [rows x 1024] bf16 arena, 2 KB row pitch, SW128) with
// different TMA box shapes / issuing threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1712_04048_b200/csrc tools/tma_tile.cu -o tools/tma_tile -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cstdio>

#include "ptx.cuh"

using namespace cavs;
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// mode 0: one 3D box {64, NT, 8}; 1: 8 2D boxes {64, NT} from one thread; 2: 8 2D boxes from 8
// warps; 3: 8 2D boxes from 8 lanes of warp 0.  reps tiles in sequence (each waits for the last).
__global__ void k_tile(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap m2, int nt, int mode,
                       int reps, int rows, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); ptx::tma_prefetch(&m3); ptx::tma_prefetch(&m2); }
  __syncthreads();
  const uint32_t bytes = nt * 128 * 8;
  unsigned long long tsum = 0;
  for (int r = 0; r < reps; ++r) {
    const int row = ((blockIdx.x * 131 + r * 977) * 64) % (rows - 4096 - 64);
    __syncthreads();
    const unsigned long long t0 = gt();
    if (threadIdx.x == 0) ptx::mbar_arrive_expect_tx(&bar, mode == 4 ? 2 * bytes : bytes);
    __syncthreads();
    if (mode == 0) {
      if (threadIdx.x == 0) ptx::tma_load_3d(smem, &m3, 0, row, 0, &bar);
    } else if (mode == 1) {
      if (threadIdx.x == 0)
        for (int kb = 0; kb < 8; ++kb) ptx::tma_load_2d(smem + kb * nt * 128, &m2, kb * 64, row, &bar);
    } else if (mode == 4) {   // two 3D boxes (two segments), issued by two warps at once
      if (lane == 0 && warp < 2) ptx::tma_load_3d(smem + warp * nt * 1024, &m3, 0, row + warp * 4096, 0, &bar);
    } else if (mode == 2) {
      if (lane == 0 && warp < 8) ptx::tma_load_2d(smem + warp * nt * 128, &m2, warp * 64, row, &bar);
    } else {
      if (warp == 0 && lane < 8) ptx::tma_load_2d(smem + lane * nt * 128, &m2, lane * 64, row, &bar);
    }
    ptx::mbar_wait(&bar, r & 1);
    tsum += gt() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tsum / reps;
}

// Written-then-read: CTA b first stores (generic st.global, like the level epilogue) the rows
// that CTA (b+1) % grid then loads by one 3D TMA box after a grid barrier.
template <int NT>
__global__ void k_wr2(const __grid_constant__ CUtensorMap m3, __nv_bfloat16* arena, int reps, int rows, unsigned* sync,
                      unsigned long long* out, int write) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); ptx::tma_prefetch(&m3); }
  __syncthreads();
  unsigned long long tsum = 0;
  for (int r = 0; r < reps; ++r) {
    const int wr = ((((blockIdx.x + 1) % gridDim.x) * 131 + r * 977) * 64) % (rows - 64);
    const int rd = ((blockIdx.x * 131 + r * 977) * 64) % (rows - 64);
    if (write) {   // the rows CTA (b+1) will read: NT rows x 512 bf16 (k-blocks 0..7), 8-byte stores
      for (int e = threadIdx.x; e < NT * 128; e += blockDim.x) {
        const int row = e / 128, c = (e % 128) * 4;
        *reinterpret_cast<uint2*>(arena + (size_t)(wr + row) * 1024 + c) = make_uint2(r, blockIdx.x);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(sync, 1u);
      const unsigned target = (r + 1) * gridDim.x;
      while ((int)(ptx::ld_acquire_gpu(sync) - target) < 0) { }
    }
    __syncthreads();
    const unsigned long long t0 = gt();
    if (threadIdx.x == 0) {
      ptx::fence_proxy_async_global();
      ptx::mbar_arrive_expect_tx(&bar, NT * 128 * 8);
      ptx::tma_load_3d(smem, &m3, 0, rd, 0, &bar);
    }
    ptx::mbar_wait(&bar, r & 1);
    tsum += gt() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tsum / reps;
}

// TMA latency of one 16 KB 3D box on CTA 0..15 while the rest of the machine generates noise:
// noise 0: none; 1: 3 warps of every CTA spin on a volatile smem word; 2: every CTA >= 16 polls
// a global counter with ld.acquire.gpu (the grid barrier's poll); 3: both.
__global__ void k_noise(const __grid_constant__ CUtensorMap m3, int reps, int rows, unsigned* flag,
                        unsigned long long* out, int noise) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); ptx::tma_prefetch(&m3); stop = 0; }
  __syncthreads();
  const bool worker = blockIdx.x < 16;
  if (warp >= 1 && warp <= 3 && lane == 0 && (noise & 1)) {
    while (!stop) { }
  } else if (warp == 0 && lane == 0) {
    if (worker) {
      unsigned long long tsum = 0;
      for (int r = 0; r < reps; ++r) {
        const int row = noise >= 4 ? ((r * 977) * 64) % (rows - 64) : ((blockIdx.x * 131 + r * 977) * 64) % (rows - 64);
        if (noise >= 4) {   // all 16 worker CTAs load the SAME rows, roughly at the same time
          if (blockIdx.x == 0) atomicAdd(flag + 8, 1u);
          while ((int)(ptx::ld_acquire_gpu(flag + 8) - (unsigned)(r + 1)) < 0) { }
        }
        const unsigned long long t0 = gt();
        ptx::mbar_arrive_expect_tx(&bar, 16 * 128 * 8);
        ptx::tma_load_3d(smem, &m3, 0, row, 0, &bar);
        ptx::mbar_wait(&bar, r & 1);
        tsum += gt() - t0;
      }
      out[blockIdx.x] = tsum / reps;
      atomicAdd(flag, 1u);
    } else if (noise & 2) {
      while (ptx::ld_acquire_gpu(flag) < 16u) { }
    }
    stop = 1;
  }
  __syncthreads();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

int main() {
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int rows = 1 << 14, width = 1024;             // 32 MB arena (L2-resident after a warm pass)
  void* buf;
  cudaMalloc(&buf, (size_t)rows * width * 2);
  cudaMemset(buf, 1, (size_t)rows * width * 2);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 148 * 8);
  cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  {
    unsigned* sync;
    cudaMalloc(&sync, 64);
    CUtensorMap m3;
    cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)width / 64};
    cuuint64_t s3[2] = {(cuuint64_t)width * 2, 128};
    cuuint32_t b3[3] = {64, 16, 8};
    cuuint32_t e3[3] = {1, 1, 1};
    enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_wr2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_noise, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int noise : {0, 4}) {
      cudaMemset(sync, 0, 64);
      k_noise<<<144, 384, 200 * 1024>>>(m3, 64, rows, sync, d_out, noise);
      cudaDeviceSynchronize();
      unsigned long long h[16];
      cudaMemcpy(h, d_out, 16 * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 16; ++i) avg += h[i];
      printf("noise %d (1: smem spin warps, 2: global acquire pollers): %6.2f us per 16 KB box  %s\n", noise,
             avg / 16 / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    for (int write : {0, 1}) {
      for (int grid : {16, 144}) {
        cudaMemset(sync, 0, 64);
        k_wr2<16><<<grid, 256, 200 * 1024>>>(m3, (__nv_bfloat16*)buf, 32, rows, sync, d_out, write);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
        double avg = 0, mx = 0;
        for (int i = 0; i < grid; ++i) { avg += h[i]; mx = h[i] > mx ? h[i] : mx; }
        avg /= grid;
        printf("after grid barrier, rows %s: grid %3d : %6.2f us avg, %6.2f max per 16 KB box  %s\n",
               write ? "WRITTEN by another SM just before" : "not written", grid, avg / 1e3, mx / 1e3,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  for (int nt : {16, 32, 64}) {
    CUtensorMap m3, m2;
    cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)width / 64};
    cuuint64_t s3[2] = {(cuuint64_t)width * 2, 128};
    cuuint32_t b3[3] = {64, (cuuint32_t)nt, 8};
    cuuint32_t e3[3] = {1, 1, 1};
    CUresult r3 = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d2[2] = {(cuuint64_t)width, (cuuint64_t)rows};
    cuuint64_t s2[1] = {(cuuint64_t)width * 2};
    cuuint32_t b2[2] = {64, (cuuint32_t)nt};
    cuuint32_t e2[2] = {1, 1};
    CUresult r2 = enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r3 || r2) { printf("encode failed %d %d\n", (int)r3, (int)r2); return 1; }
    const char* names[5] = {"3D box x1, 1 thread ", "2D box x8, 1 thread ", "2D box x8, 8 warps  ", "2D box x8, 8 lanes  ",
                            "3D box x2, 2 warps   "};
    for (int mode : {0, 4}) {
      for (int grid : {1, 144}) {
        k_tile<<<grid, 256, 200 * 1024>>>(m3, m2, nt, mode, 32, rows, d_out);
        k_tile<<<grid, 256, 200 * 1024>>>(m3, m2, nt, mode, 32, rows, d_out);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < grid; ++i) avg += h[i];
        avg /= grid;
        printf("NT=%2d %s grid %3d : %6.2f us per %2d KB tile (%6.1f GB/s per SM)  %s\n", nt, names[mode], grid, avg / 1e3,
               nt * 8 * 128 / 1024, nt * 8 * 128 / avg, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
