// Micro-benchmark of the pipeline primitives used by salr_linear_kernel
// (cycles per op, one CTA): mbarrier test_wait/try_wait on a completed phase,
// arrive, arrive.expect_tx, 1-D bulk copy issue, 2-D tensor TMA issue, and a
// full producer->consumer hand-off between two warps.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2601_16991_b200/csrc/salr_ptx.cuh"
using namespace salr;

__global__ void ubench(const __grid_constant__ CUtensorMap xmap, const uint8_t* src, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    const int N = 64;
    long long t0, t1;
    // (a) test_wait on a barrier whose phase 0 is not complete -> parity 1 "previous phase" passes
    t0 = clock64();
    for (int i = 0; i < N; ++i) mbar_test_wait(&bar[0], 1);
    t1 = clock64(); out[0] = (t1 - t0) / N;
    t0 = clock64();
    for (int i = 0; i < N; ++i) mbar_try_wait(&bar[0], 1);
    t1 = clock64(); out[1] = (t1 - t0) / N;
    // (b) arrive (count 1 -> completes phase each time)
    t0 = clock64();
    for (int i = 0; i < N; ++i) mbar_arrive(&bar[1]);
    t1 = clock64(); out[2] = (t1 - t0) / N;
    // (c) arrive.expect_tx with 0 bytes
    t0 = clock64();
    for (int i = 0; i < N; ++i) mbar_arrive_expect_tx(&bar[2], 0);
    t1 = clock64(); out[3] = (t1 - t0) / N;
    // (d) bulk copy issue 4 KB each (completion on bar[3])
    mbar_arrive_expect_tx(&bar[3], 16 * 4096);
    t0 = clock64();
    for (int i = 0; i < 16; ++i) bulk_g2s(sm + (i & 7) * 4096, src + (size_t)i * 4096, 4096, &bar[3]);
    t1 = clock64(); out[4] = (t1 - t0) / 16;
    t0 = clock64();
    mbar_wait(&bar[3], 0);
    t1 = clock64(); out[5] = t1 - t0;  // latency to completion after issue
    // (e) tensor TMA issue 2 KB boxes
    mbar_arrive_expect_tx(&bar[4], 16 * 64 * 16 * 2);
    t0 = clock64();
    for (int i = 0; i < 16; ++i) tma_2d_g2s(sm + 32768 + (i & 7) * 2048, &xmap, 64 * i, 0, &bar[4]);
    t1 = clock64(); out[6] = (t1 - t0) / 16;
    t0 = clock64();
    mbar_wait(&bar[4], 0);
    t1 = clock64(); out[7] = t1 - t0;
    // (f) globaltimer read cost
    unsigned long long g;
    t0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    t1 = clock64(); out[8] = (t1 - t0) / N;
  }
  __syncthreads();
  // (g) ping-pong hand-off latency between warp 0 and warp 1 (round trip)
  if (warp < 2) {
    const int N = 64;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
      if (warp == 0) {
        if (lane == 0) mbar_arrive(&bar[5]);
        mbar_wait(&bar[6], i & 1);
      } else {
        mbar_wait(&bar[5], i & 1);
        if (lane == 0) mbar_arrive(&bar[6]);
      }
    }
    long long t1 = clock64();
    if (warp == 0 && lane == 0) out[9] = (t1 - t0) / N;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  uint8_t* src;
  cudaMalloc(&src, 1 << 24);
  cudaMemset(src, 1, 1 << 24);
  long long* out;
  cudaMalloc(&out, 64 * 8);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {4096, 64};
  cuuint64_t str[1] = {4096 * 2};
  cuuint32_t box[2] = {64, 16};
  cuuint32_t es[2] = {1, 1};
  ((EncFn)fp)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(ubench, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int rep = 0; rep < 3; ++rep) {
    ubench<<<1, 64, 70000>>>(map, src, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, out, 16 * 8, cudaMemcpyDeviceToHost);
    printf("rep %d err=%d: test_wait %lld, try_wait %lld, arrive %lld, arrive_expect_tx %lld, bulk issue %lld, "
           "bulk latency %lld, tma2d issue %lld, tma2d latency %lld, globaltimer %lld, pingpong %lld cycles\n",
           rep, (int)e, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
  }
  return 0;
}
