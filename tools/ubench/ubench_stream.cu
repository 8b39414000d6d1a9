// Micro-benchmark: HBM streaming with 1-D bulk copies into a shared-memory
// ring (the record path of the fused linear without decode or MMA).  One CTA
// per SM, one producer warp, one consumer warp that releases each stage as
// soon as it lands.  Reports achieved GB/s for ring depth x record size.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench/ubench_stream tools/ubench/ubench_stream.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2601_16991_b200/csrc/salr_ptx.cuh"
using namespace salr;

__global__ void __launch_bounds__(64, 1) stream_kernel(const uint8_t* __restrict__ src, int64_t total_units,
                                                        uint32_t rec, int S, int evict_first, int hops) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * rec);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t u0 = blockIdx.x * total_units / G, u1 = (blockIdx.x + 1) * total_units / G;
  const uint64_t pol = l2_policy_evict_first();
  if (warp == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int64_t u = u0; u < u1; ++u) {
      if (u - u0 >= S) mbar_wait(&empty[s], ph ^ 1);
      if (lane == 0) {
        if (evict_first)
          bulk_g2s_hint(sm + (size_t)s * rec, src + u * rec, rec, &full[s], pol);
        else
          bulk_g2s(sm + (size_t)s * rec, src + u * rec, rec, &full[s]);
        mbar_arrive_expect_tx(&full[s], rec);
      }
      __syncwarp();
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else {
    int s = 0;
    uint32_t ph = 0;
    uint32_t acc = 0;
    for (int64_t u = u0; u < u1; ++u) {
      mbar_wait(&full[s], ph);
      acc += *reinterpret_cast<volatile uint32_t*>(sm + (size_t)s * rec + 4 * lane);
      for (int h = 0; h < hops; ++h) __nanosleep(100);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) printf("x");
  }
}

int main() {
  const int64_t bytes_total = 4ll << 30;  // 4 GiB streamed per launch
  uint8_t* src;
  cudaMalloc(&src, bytes_total + (1 << 20));
  cudaMemset(src, 1, bytes_total);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t recs[] = {4096, 9344, 16384};
  for (int ef = 0; ef < 2; ++ef)
    for (uint32_t rec : recs)
      for (int S : {4, 8, 12, 16, 20}) {
        const size_t smem = (size_t)S * rec + 16 * S + 64;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t units = bytes_total / rec;
        stream_kernel<<<148, 64, smem>>>(src, units, rec, S, ef, 0);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) stream_kernel<<<148, 64, smem>>>(src, units, rec, S, ef, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = 3.0 * units * rec / (ms * 1e-3) / 1e9;
        printf("evict_first=%d rec=%5u S=%2d  in flight/SM=%6zu B  %7.1f GB/s\n", ef, rec, S, (size_t)S * rec, gbs);
      }
  cudaError_t err = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
