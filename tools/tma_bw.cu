// tools/tma_bw.cu — microbenchmark: per-SM TMA ingest bandwidth vs. box shape / bytes in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1712_04048_b200/csrc tools/tma_bw.cu -o tools/tma_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace cavs;
__device__ __forceinline__ unsigned long long gtime_dev() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// mode 1: batch-issue `inflight` boxes then wait for all; mode 2: `inflight` warps each issue their own stream
__global__ void k_tma2(const __grid_constant__ CUtensorMap m, int box_rows, int nboxes, int inflight, int rows_total,
                       unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  const int box_bytes = 128 * box_rows;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long t0 = gtime_dev();
  const int row0 = (blockIdx.x * 977) % (rows_total - box_rows);
  if (mode == 1) {
    if (threadIdx.x == 0) {
      uint32_t phase = 0;
      for (int b0 = 0; b0 < nboxes; b0 += inflight) {
        for (int i = 0; i < inflight; ++i) {
          ptx::mbar_arrive_expect_tx(&bar[i], box_bytes);
          ptx::tma_load_2d(smem + i * box_bytes, &m, 0, (row0 + (b0 + i) * box_rows) % (rows_total - box_rows), &bar[i]);
        }
        for (int i = 0; i < inflight; ++i) ptx::mbar_wait(&bar[i], phase);
        phase ^= 1;
      }
    }
  } else {
    const int w = threadIdx.x >> 5;
    if (w < inflight && (threadIdx.x & 31) == 0) {
      uint32_t phase = 0;
      for (int b = w; b < nboxes; b += inflight) {
        ptx::mbar_arrive_expect_tx(&bar[w], box_bytes);
        ptx::tma_load_2d(smem + w * box_bytes, &m, 0, (row0 + b * box_rows) % (rows_total - box_rows), &bar[w]);
        ptx::mbar_wait(&bar[w], phase);
        phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = gtime_dev() - t0;
}

__global__ void k_tma(const __grid_constant__ CUtensorMap m, int box_rows, int nboxes, int inflight, int rows_total,
                      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  const int box_bytes = 128 * box_rows;
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t0 = gtime_dev();
    int issued = 0, done = 0;
    uint32_t phase[16] = {0};
    const int row0 = (blockIdx.x * 977) % (rows_total - box_rows);
    while (done < nboxes) {
      while (issued < nboxes && issued - done < inflight) {
        const int s = issued % inflight;
        ptx::mbar_arrive_expect_tx(&bar[s], box_bytes);
        ptx::tma_load_2d(smem + s * box_bytes, &m, 0, (row0 + issued * box_rows) % (rows_total - box_rows), &bar[s]);
        ++issued;
      }
      const int s = done % inflight;
      ptx::mbar_wait(&bar[s], phase[s]);
      phase[s] ^= 1;
      ++done;
    }
    out[blockIdx.x] = gtime_dev() - t0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

int main() {
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int rows = 1 << 16, cols = 64;                      // 64 bf16 = 128 B rows, 8 MB total (L2-resident)
  void* buf;
  cudaMalloc(&buf, (size_t)rows * 1024);
  cudaMemset(buf, 1, (size_t)rows * 1024);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 148 * 8);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_tma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode : {1, 2}) {
    for (int box_rows : {64, 128, 256}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {64, (cuuint64_t)rows};
      cuuint64_t strides[1] = {1024};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int inflight : {1, 2, 4, 8}) {
        if (inflight * 128 * box_rows > 196 * 1024) continue;
        const int nboxes = (4 << 20) / (128 * box_rows);
        for (int rep = 0; rep < 2; ++rep)
          k_tma2<<<16, 32 * 8, inflight * 128 * box_rows>>>(m, box_rows, nboxes, inflight, rows, d_out, mode);
        cudaDeviceSynchronize();
        unsigned long long t[16];
        cudaMemcpy(t, d_out, 16 * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (auto v : t) mx = v > mx ? v : mx;
        printf("mode %d box_rows %3d inflight %d grid 16 : %7.1f GB/s per CTA\n", mode, box_rows, inflight,
               (4 << 20) / (double)mx);
      }
    }
  }
  for (int pitch_el : {512}) {
    for (int box_rows : {64, 128, 256}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)pitch_el * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int inflight : {1, 2, 4, 8, 12}) {
        if (inflight * 128 * box_rows > 196 * 1024) continue;
        for (int grid : {1, 16, 148}) {
          const int nboxes = (4 << 20) / (128 * box_rows);  // 4 MB per CTA
          for (int rep = 0; rep < 2; ++rep)
            k_tma<<<grid, 32, inflight * 128 * box_rows>>>(m, box_rows, nboxes, inflight, rows, d_out);
          cudaDeviceSynchronize();
          std::vector<unsigned long long> t(grid);
          cudaMemcpy(t.data(), d_out, grid * 8, cudaMemcpyDeviceToHost);
          unsigned long long mx = 0;
          for (auto v : t) mx = v > mx ? v : mx;
          printf("pitch %4dB box_rows %3d inflight %2d (%6.1f KB) grid %3d : %7.1f GB/s per CTA, %8.1f GB/s total\n",
                 pitch_el * 2, box_rows, inflight, inflight * 128 * box_rows / 1024.0, grid,
                 (4 << 20) / (double)mx, (double)grid * (4 << 20) / (double)mx);
        }
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
