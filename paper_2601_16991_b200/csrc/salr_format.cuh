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

// TB2: the linear kernel's compute format, built once per matrix from bf16
// TB records (salr_tb2_*).  Same tile grid, same logical content; per tile:
//   u32 hdr[4]           value offsets of groups 1,2,3 and the tile nnz
//   u16 bandoff[4][16]   per 32-column group g and 4-row band b: offset of the
//                        band's values from the group's first value
//   u64 cmask[128]       cmask[n] bit r <=> element (row r, col n) nonzero
//   bf16 values          group-major; within a group band-major; within a band
//                        column-major; within a column ascending rows
// so a decoder lane (one output column) finds its band's values contiguous.
constexpr int kT2BandOff = 16;
constexpr int kT2Mask = 144;
constexpr int kT2Val = 1168;
constexpr int kMaxRecordBytesT2 = kT2Val + kTileK * kTileN * 2;  // 17552

// NM24: compute format of a matrix whose nonzeros are 2:4 along the columns
// (at most 2 in every group of 4 consecutive columns of a row -- the
// reference's N:M mask, prune.py:238-248).  Fixed 9216 bytes per 64x128 tile,
// n-tile-major like TB2 (no offset table: tile t starts at 9216 * t):
//   values  [16 bands][32 groups] x 16 B: for the 4 rows of the band one u32
//           each, v0 | v1 << 16 = the group's first and second nonzero (bf16;
//           0 when absent), at 16 * (32 * band + group)
//   masks   [2 halves][32 groups] x 16 B at 8192: u32 word w of (half h,
//           group g) holds rows 32h + 8w .. +7, row i's 4-bit column mask
//           (bit j = column 4g + j nonzero) at bits 4i .. 4i+3
// 1.125 B/weight; a decoder lane selects its column's value of each row with
// byte permutes -- no prefix sums, no variable offsets.
constexpr int kNmValBytes = 8192;
constexpr int kNmRecBytes = 9216;

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
