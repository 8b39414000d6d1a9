// Micro-benchmark: tcgen05.mma (kind::f16, M=128, K=16) issue cost for small N,
// A operand from TMEM (ts) or SMEM (ss); commit + wait latency.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2601_16991_b200/csrc/salr_ptx.cuh"
using namespace salr;

template <int N>
__global__ void ubench(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536 + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  constexpr uint32_t IDESC = idesc_bf16_f32(128, N);
  if (warp == 0 && lane == 0) {
    const uint64_t bdesc = desc_kmajor_sw128(smem_u32(sm));
    const uint64_t adesc = desc_kmajor_sw128(smem_u32(sm + 32768));
    long long t0, t1;
    const int R = 64;
    // ts: 4 MMAs (K=64) per "unit", then commit, repeated R times (no waits)
    t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_ts(tmem, tmem + 256 + 8 * j, bdesc + 2 * j, IDESC, 1u);
      tc_commit(&bar[0]);
    }
    t1 = clock64();
    out[0] = (t1 - t0) / R;  // issue cost per unit (4 mma + commit)
    t0 = clock64();
    mbar_wait(&bar[0], (R - 1) & 1);
    t1 = clock64();
    out[1] = t1 - t0;  // drain
    // ss variant
    t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_ss(tmem, adesc + 2 * j, bdesc + 2 * j, IDESC, 1u);
      tc_commit(&bar[1]);
    }
    t1 = clock64();
    out[2] = (t1 - t0) / R;
    t0 = clock64();
    mbar_wait(&bar[1], (R - 1) & 1);
    t1 = clock64();
    out[3] = t1 - t0;
    // ts without per-unit commit (one commit at the end)
    t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_ts(tmem, tmem + 256 + 8 * j, bdesc + 2 * j, IDESC, 1u);
    }
    tc_commit(&bar[3]);
    t1 = clock64();
    out[5] = (t1 - t0) / R;
    // commit only
    t0 = clock64();
    for (int r = 0; r < R; ++r) tc_commit(&bar[3]);
    t1 = clock64();
    out[6] = (t1 - t0) / R;
    out[7] = 0;
    // serial: unit = 4 mma + commit + wait for completion (latency per unit)
    t0 = clock64();
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_ts(tmem, tmem + 256 + 8 * j, bdesc + 2 * j, IDESC, 1u);
      tc_commit(&bar[2]);
      mbar_wait(&bar[2], r & 1);
    }
    t1 = clock64();
    out[4] = (t1 - t0) / 16;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 64 * 8);
  cudaFuncSetAttribute(ubench<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(ubench<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(ubench<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int rep = 0; rep < 2; ++rep) {
    long long h[8];
    ubench<16><<<1, 128, 70000>>>(out);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, 8 * 8, cudaMemcpyDeviceToHost);
    printf("N=16 err=%d: ts unit issue %lld, drain %lld | ss unit issue %lld, drain %lld | serial unit %lld cycles | 4mma no commit %lld | commit %lld | ktile_ts %lld\n",
           (int)e, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    ubench<32><<<1, 128, 70000>>>(out);
    e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, 8 * 8, cudaMemcpyDeviceToHost);
    printf("N=32 err=%d: ts unit issue %lld, drain %lld | ss unit issue %lld, drain %lld | serial unit %lld cycles\n",
           (int)e, h[0], h[1], h[2], h[3], h[4]);
    ubench<128><<<1, 128, 70000>>>(out);
    e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, 8 * 8, cudaMemcpyDeviceToHost);
    printf("N=128 err=%d: ts unit issue %lld, drain %lld | ss unit issue %lld, drain %lld | serial unit %lld cycles\n",
           (int)e, h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
