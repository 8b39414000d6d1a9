// TB ("tiled bitmap") record format shared by the codec and the linear kernels.
// See include/salr_b200.h for the byte layout.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace salr {

constexpr int kTileK = 64;          // rows (d_in / K) per tile
constexpr int kTileN = 128;         // cols (d_out / N) per tile
constexpr int kGroups = 4;          // 32-column groups per tile
constexpr int kHdrBytes = 16;       // u32 hdr[4]
constexpr int kBitsBytes = kGroups * kTileK * 4;      // 1024
constexpr int kValOffset = kHdrBytes + kBitsBytes;    // 1040
constexpr int kMaxRecordBytesBf16 = kValOffset + kTileK * kTileN * 2;  // 17424

enum : int { kF32 = 0, kBF16 = 1, kF64 = 2 };

__host__ __device__ inline int value_bytes(int dtype) { return dtype == kF32 ? 4 : 2; }

// Record size in 16-byte units for a tile holding nnz values of vbytes each.
__host__ __device__ inline uint32_t record_units(uint32_t nnz, int vbytes) {
  uint32_t bytes = kValOffset + nnz * (uint32_t)vbytes;
  return (bytes + 15u) / 16u;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Load element i of a dense matrix of the given dtype as float32 (RN for f64).
__device__ __forceinline__ float load_as_f32(const void* p, int dtype, int64_t i) {
  if (dtype == kF32) return static_cast<const float*>(p)[i];
  if (dtype == kBF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __double2float_rn(static_cast<const double*>(p)[i]);
}

}  // namespace salr
