// Micro-benchmark of the fused linear's MMA-issue loop (one converged warp,
// one elected lane issuing): cycles per unit for 4 x tcgen05.mma (M=128,
// N=16, K=16, A in TMEM) + commit, with the kernel's operand bookkeeping,
// against variants with fewer uniform-register moves.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench/ubench_mma2 tools/ubench/ubench_mma2.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2601_16991_b200/csrc/salr_ptx.cuh"
using namespace salr;

constexpr int kS = 8;
constexpr uint32_t kN = KN;

// 4 MMAs with immediate TMEM/descriptor offsets from one base per operand.
__device__ __forceinline__ void mma_ktile_imm(uint32_t d_tm, uint32_t a_tm, uint64_t bdesc, uint32_t idesc,
                                              uint32_t acc, uint32_t empty_bar) {
  asm volatile(
      "{\n\t.reg .pred pe, pa;\n\t"
      ".reg .b64 d1, d2, d3;\n\t"
      ".reg .b32 a1, a2, a3;\n\t"
      "elect.sync _|pe, 0xffffffff;\n\t"
      "setp.ne.b32 pa, %4, 0;\n\t"
      "add.s64 d1, %2, 2;\n\t"
      "add.s64 d2, %2, 4;\n\t"
      "add.s64 d3, %2, 6;\n\t"
      "add.u32 a1, %1, 8;\n\t"
      "add.u32 a2, %1, 16;\n\t"
      "add.u32 a3, %1, 24;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, pa;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], d1, %3, 1;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], d2, %3, 1;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], d3, %3, 1;\n\t"
      "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(d_tm),
      "r"(a_tm), "l"(bdesc), "r"(idesc), "r"(acc), "r"(empty_bar)
      : "memory");
}

__global__ void bench(long long* out, int R) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kS + 2; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t IDESC = idesc_bf16_f32(128, kN);
  if (warp == 0) {
    const uint64_t bdesc0 = desc_kmajor_sw128(smem_u32(sm));
    const uint32_t lo0 = (uint32_t)bdesc0, hi = (uint32_t)(bdesc0 >> 32);
    constexpr uint32_t kLoStep = (kN * 128) >> 4;
    long long t0, t1;
    // (a) kernel form: incremental stage addresses, ktile asm block, commit per unit
    {
      uint32_t lo = lo0, atm = 64, ead = smem_u32(&bar[0]);
      int s = 0;
      __syncwarp();
      t0 = clock64();
      for (int v = 0; v < R; ++v) {
        mma_ktile_ts(tmem, atm, lo, hi, IDESC, v != 0, ead);
        if (++s == kS) { s = 0; lo = lo0; atm = 64; ead = smem_u32(&bar[0]); }
        else { lo += kLoStep; atm += 32; ead += 8; }
      }
      __syncwarp();
      t1 = clock64();
      if (threadIdx.x == 0) out[0] = (t1 - t0) / R;
      // execution throughput: wait for the last unit's commit
      if (elect_one()) tc_commit(&bar[2 * kS]);
      __syncwarp();
      mbar_wait(&bar[2 * kS], 0);
      const long long t2 = clock64();
      if (threadIdx.x == 0) out[4] = (t2 - t0) / R;
    }
    // (b) unrolled by the ring depth: compile-time stage offsets
    {
      __syncwarp();
      t0 = clock64();
      for (int v = 0; v < R; v += kS) {
#pragma unroll
        for (int s = 0; s < kS; ++s)
          mma_ktile_imm(tmem, 64 + 32 * s, bdesc0 + s * kLoStep, IDESC, 1, smem_u32(&bar[s]));
      }
      __syncwarp();
      t1 = clock64();
      if (threadIdx.x == 0) out[1] = (t1 - t0) / R;
    }
    // (c) like (b) plus the kernel's per-unit waits: try_wait on a completed
    // barrier, fence, probe of the next barrier
    {
      const uint32_t done = smem_u32(&bar[2 * kS + 1]);
      if (threadIdx.x == 0) mbar_arrive(&bar[2 * kS + 1]);
      __syncwarp();
      t0 = clock64();
      for (int v = 0; v < R; v += kS) {
#pragma unroll
        for (int s = 0; s < kS; ++s) {
          mbar_wait_addr(done, 0);
          mbar_wait_addr(done, 0);
          tc_fence_after();
          const bool nr = __any_sync(0xffffffffu, mbar_test_addr(done, 0));
          mma_ktile_imm(tmem, 64 + 32 * s, bdesc0 + s * kLoStep, IDESC, nr ? 1u : 1u, smem_u32(&bar[s]));
        }
      }
      __syncwarp();
      t1 = clock64();
      if (threadIdx.x == 0) out[2] = (t1 - t0) / R;
    }
    // (d) MMAs only, no commits
    {
      __syncwarp();
      t0 = clock64();
      for (int v = 0; v < R; ++v) {
        if (elect_one()) {
#pragma unroll
          for (int j = 0; j < 4; ++j) mma_ts(tmem, 64 + 32 * (v & 7) + 8 * j, bdesc0 + 2 * j, IDESC, 1u);
        }
        __syncwarp();
      }
      t1 = clock64();
      if (threadIdx.x == 0) out[3] = (t1 - t0) / R;
      if (elect_one()) tc_commit(&bar[2 * kS]);
      __syncwarp();
      mbar_wait(&bar[2 * kS], 1);
    }
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
  cudaMalloc(&out, 16 * 8);
  cudaMemset(out, 0, 16 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int rep = 0; rep < 3; ++rep) {
    long long h[5];
    bench<<<1, 128, 70000>>>(out, 256);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, 5 * 8, cudaMemcpyDeviceToHost);
    printf("err=%d cycles/unit: kernel-form issue %lld, executed %lld | unrolled imm %lld | +waits/probe %lld | mma only %lld\n",
           (int)e, h[0], h[4], h[1], h[2], h[3]);
  }
  return 0;
}
