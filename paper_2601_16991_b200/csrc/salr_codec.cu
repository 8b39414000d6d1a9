// Bitmap codec kernels for the TB tile format: encode (two-pass, warp-ballot /
// popc prefix offsets), decode / decode-window, and bit-exact conversion to
// and from the reference's row-major bitmap + value layout.
//
// Reference semantics restated here:
//   encode        pkg/src/salr/bitmap.py:150-165  (f32 cast, +0.0, != 0 mask,
//                 LSB-first packing, row-major value order)
//   decode        pkg/src/salr/bitmap.py:168-180
//   decode_block  pkg/src/salr/bitmap.py:183-212
//   storage       pkg/src/salr/bitmap.py:88-143   (bitmap rows x ceil(cols/8))
#include <cstdint>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "salr_format.cuh"
#include "salr_status.cuh"

namespace salr {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// ------------------------------------------------------------------ scans
// Single-block exclusive scan of n u32 items produced by a functor; writes
// out[0..n] (out[n] = total).  Used for tile and row-tile offsets (setup-time
// work; n <= a few million).
struct TileUnitsFn {
  const uint32_t* cnt;
  int vbytes;
  __device__ uint32_t operator()(int64_t t) const {
    uint32_t c = cnt[4 * t] + cnt[4 * t + 1] + cnt[4 * t + 2] + cnt[4 * t + 3];
    return record_units(c, vbytes);
  }
};
struct ArrayFn {
  const uint32_t* a;
  __device__ uint32_t operator()(int64_t i) const { return a[i]; }
};

template <class F>
__global__ void __launch_bounds__(1024) scan1_kernel(F f, int64_t n, uint32_t* out) {
  constexpr int kItems = 4;
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += 1024 * kItems) {
    uint32_t v[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      int64_t idx = base + (int64_t)tid * kItems + i;
      v[i] = idx < n ? f(idx) : 0u;
      sum += v[i];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = warp_tot[lane];
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      warp_tot[lane] = wi - w;  // exclusive
    }
    __syncthreads();
    uint32_t run = carry_s + warp_tot[warp] + incl - sum;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      int64_t idx = base + (int64_t)tid * kItems + i;
      if (idx < n) out[idx] = run;
      run += v[i];
    }
    __syncthreads();
    if (tid == 1023) carry_s = run;
    __syncthreads();
  }
  if (tid == 0) out[n] = carry_s;
}

// ------------------------------------------------------------------ encode
// grid = n_tiles, block = 128 (warp g <-> 32-column group g, lane <-> column).
__global__ void encode_count_kernel(const void* __restrict__ dense, int in_dtype, int64_t rows,
                                    int64_t cols, int64_t ld, int64_t n_kt,
                                    uint32_t* __restrict__ tile_cnt) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col = nt * kTileN + 32 * g + lane;
  uint32_t cnt = 0;
  for (int k = 0; k < kTileK; ++k) {
    const int64_t row = kt * kTileK + k;
    bool keep = false;
    if (row < rows && col < cols) keep = load_as_f32(dense, in_dtype, row * ld + col) != 0.0f;
    cnt += __popc(__ballot_sync(0xffffffffu, keep));
  }
  if (lane == 0) tile_cnt[4 * t + g] = cnt;
}

__global__ void encode_write_kernel(const void* __restrict__ dense, int in_dtype, int64_t rows,
                                    int64_t cols, int64_t ld, int64_t n_kt, int value_dtype,
                                    const uint32_t* __restrict__ tile_cnt,
                                    const uint32_t* __restrict__ tile_off,
                                    uint8_t* __restrict__ records) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col = nt * kTileN + 32 * g + lane;
  uint8_t* rec = records + 16ull * tile_off[t];
  uint32_t* hdr = reinterpret_cast<uint32_t*>(rec);
  uint32_t* bits = hdr + 4;
  const uint32_t c0 = tile_cnt[4 * t], c1 = tile_cnt[4 * t + 1], c2 = tile_cnt[4 * t + 2],
                 c3 = tile_cnt[4 * t + 3];
  const uint32_t gbase[4] = {0u, c0, c0 + c1, c0 + c1 + c2};
  const uint32_t nnz = c0 + c1 + c2 + c3;
  if (threadIdx.x == 0) {
    hdr[0] = gbase[1];
    hdr[1] = gbase[2];
    hdr[2] = gbase[3];
    hdr[3] = nnz;
  }
  const uint32_t lt = lanemask_lt();
  uint32_t off = gbase[g];
  const int vb = value_bytes(value_dtype);
  for (int k = 0; k < kTileK; ++k) {
    const int64_t row = kt * kTileK + k;
    float f = 0.0f;
    if (row < rows && col < cols) f = load_as_f32(dense, in_dtype, row * ld + col) + 0.0f;
    const bool keep = f != 0.0f;
    const uint32_t word = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) bits[g * kTileK + k] = word;
    if (keep) {
      const uint32_t idx = off + __popc(word & lt);
      if (value_dtype == kBF16)
        reinterpret_cast<__nv_bfloat16*>(rec + kValOffset)[idx] = __float2bfloat16_rn(f);
      else
        reinterpret_cast<float*>(rec + kValOffset)[idx] = f;
    }
    off += __popc(word);
  }
  // zero the pad bytes up to the 16-byte record boundary
  if (threadIdx.x < 16) {
    const uint32_t used = kValOffset + nnz * vb;
    const uint32_t end = 16u * (tile_off[t + 1] - tile_off[t]);
    const uint32_t b = used + threadIdx.x;
    if (b < end) rec[b] = 0;
  }
}

// ------------------------------------------------------------------ decode
__device__ __forceinline__ float tb_value(const uint8_t* rec, int value_dtype, uint32_t idx) {
  if (value_dtype == kBF16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(rec + kValOffset)[idx]);
  return reinterpret_cast<const float*>(rec + kValOffset)[idx];
}

__global__ void decode_kernel(const uint8_t* __restrict__ records, const uint32_t* __restrict__ tile_off,
                              int value_dtype, int64_t n_kt, int64_t r0, int64_t r1, int64_t c0,
                              int64_t c1, int64_t kt0, int64_t nt0, int64_t kt_span, void* out,
                              int out_dtype, int64_t ld_out) {
  const int64_t kt = kt0 + blockIdx.x % kt_span;
  const int64_t nt = nt0 + blockIdx.x / kt_span;
  const int64_t t = nt * n_kt + kt;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col = nt * kTileN + 32 * g + lane;
  const uint8_t* rec = records + 16ull * tile_off[t];
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec);
  const uint32_t* bits = hdr + 4 + g * kTileK;
  uint32_t off = g == 0 ? 0u : hdr[g - 1];
  const uint32_t lt = lanemask_lt();
  const bool col_in = col >= c0 && col < c1;
  for (int k = 0; k < kTileK; ++k) {
    const int64_t row = kt * kTileK + k;
    const uint32_t word = bits[k];
    if (col_in && row >= r0 && row < r1) {
      float v = 0.0f;
      if ((word >> lane) & 1u) v = tb_value(rec, value_dtype, off + __popc(word & lt));
      const int64_t o = (row - r0) * ld_out + (col - c0);
      if (out_dtype == kF32) static_cast<float*>(out)[o] = v;
      else if (out_dtype == kBF16) static_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(v);
      else static_cast<double*>(out)[o] = (double)v;
    }
    off += __popc(word);
  }
}

__global__ void tb_nnz_kernel(const uint8_t* __restrict__ records, const uint32_t* __restrict__ tile_off,
                              int64_t n_tiles, unsigned long long* nnz) {
  unsigned long long s = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
       t += (int64_t)gridDim.x * blockDim.x)
    s += reinterpret_cast<const uint32_t*>(records + 16ull * tile_off[t])[3];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(nnz, s);
}

// ------------------------------------------------------------------ TB -> reference
// rowtile_cnt[row * n_nt + nt] = set bits of `row` inside tile column nt.
__global__ void tb_rowtile_count_kernel(const uint8_t* __restrict__ records,
                                        const uint32_t* __restrict__ tile_off, int64_t rows,
                                        int64_t n_kt, int64_t n_nt, uint32_t* __restrict__ cnt) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int k = threadIdx.x;  // 64 threads
  const int64_t row = kt * kTileK + k;
  if (row >= rows) return;
  const uint32_t* bits = reinterpret_cast<const uint32_t*>(records + 16ull * tile_off[t]) + 4;
  uint32_t c = 0;
#pragma unroll
  for (int g = 0; g < kGroups; ++g) c += __popc(bits[g * kTileK + k]);
  cnt[row * n_nt + nt] = c;
}

__global__ void tb_to_reference_kernel(const uint8_t* __restrict__ records,
                                       const uint32_t* __restrict__ tile_off, int value_dtype,
                                       int64_t rows, int64_t cols, int64_t n_kt, int64_t n_nt,
                                       const uint32_t* __restrict__ rowtile_off,
                                       uint8_t* __restrict__ bitmap_out, void* values_out,
                                       int values_dtype) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bpr = (cols + 7) / 8;
  const uint8_t* rec = records + 16ull * tile_off[t];
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec);
  const uint32_t* bits = hdr + 4;
  uint32_t off = g == 0 ? 0u : hdr[g - 1];
  const uint32_t lt = lanemask_lt();
  for (int k = 0; k < kTileK; ++k) {
    const int64_t row = kt * kTileK + k;
    const uint32_t word = bits[g * kTileK + k];
    if (row < rows) {
      uint32_t before = 0;
      for (int gg = 0; gg < g; ++gg) before += __popc(bits[gg * kTileK + k]);
      if ((word >> lane) & 1u) {
        const float v = tb_value(rec, value_dtype, off + __popc(word & lt));
        const uint32_t ridx = rowtile_off[row * n_nt + nt] + before + __popc(word & lt);
        if (values_dtype == kF32) static_cast<float*>(values_out)[ridx] = v;
        else static_cast<__nv_bfloat16*>(values_out)[ridx] = __float2bfloat16_rn(v);
      }
      if (lane < 4) {
        const int64_t cb = nt * 16 + 4 * g + lane;
        if (cb < bpr) bitmap_out[row * bpr + cb] = (uint8_t)(word >> (8 * lane));
      }
    }
    off += __popc(word);
  }
}

// ------------------------------------------------------------------ reference -> TB
__device__ __forceinline__ uint32_t ref_word(const uint8_t* __restrict__ bitmap, int64_t bpr,
                                             int64_t row, int64_t byte0) {
  uint32_t w = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t b = byte0 + j;
    if (b < bpr) w |= (uint32_t)bitmap[row * bpr + b] << (8 * j);
  }
  return w;
}

__global__ void ref_rowtile_count_kernel(const uint8_t* __restrict__ bitmap, int64_t rows, int64_t cols,
                                         int64_t n_nt, uint32_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * n_nt) return;
  const int64_t row = i / n_nt, nt = i % n_nt;
  const int64_t bpr = (cols + 7) / 8;
  uint32_t c = 0;
#pragma unroll
  for (int g = 0; g < kGroups; ++g) c += __popc(ref_word(bitmap, bpr, row, nt * 16 + 4 * g));
  cnt[i] = c;
}

// tile_cnt[4t+g] from the reference bitmap; one thread per (tile, group).
__global__ void ref_tile_count_kernel(const uint8_t* __restrict__ bitmap, int64_t rows, int64_t cols,
                                      int64_t n_kt, int64_t n_tiles, uint32_t* __restrict__ tile_cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_tiles * kGroups) return;
  const int64_t t = i / kGroups;
  const int g = (int)(i % kGroups);
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int64_t bpr = (cols + 7) / 8;
  uint32_t c = 0;
  for (int k = 0; k < kTileK; ++k) {
    const int64_t row = kt * kTileK + k;
    if (row < rows) c += __popc(ref_word(bitmap, bpr, row, nt * 16 + 4 * g));
  }
  tile_cnt[i] = c;
}

__global__ void ref_to_tb_kernel(const uint8_t* __restrict__ bitmap, const void* values, int values_dtype,
                                 int64_t rows, int64_t cols, int64_t n_kt, int64_t n_nt, int value_dtype,
                                 const uint32_t* __restrict__ rowtile_off,
                                 const uint32_t* __restrict__ tile_cnt,
                                 const uint32_t* __restrict__ tile_off, uint8_t* __restrict__ records) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bpr = (cols + 7) / 8;
  uint8_t* rec = records + 16ull * tile_off[t];
  uint32_t* hdr = reinterpret_cast<uint32_t*>(rec);
  uint32_t* bits = hdr + 4;
  const uint32_t c0 = tile_cnt[4 * t], c1 = tile_cnt[4 * t + 1], c2 = tile_cnt[4 * t + 2],
                 c3 = tile_cnt[4 * t + 3];
  const uint32_t gbase[4] = {0u, c0, c0 + c1, c0 + c1 + c2};
  const uint32_t nnz = c0 + c1 + c2 + c3;
  if (threadIdx.x == 0) {
    hdr[0] = gbase[1];
    hdr[1] = gbase[2];
    hdr[2] = gbase[3];
    hdr[3] = nnz;
  }
  const uint32_t lt = lanemask_lt();
  uint32_t off = gbase[g];
  for (int k = 0; k < kTileK; ++k) {
    const int64_t row = kt * kTileK + k;
    uint32_t word = 0, before = 0;
    if (row < rows) {
      for (int gg = 0; gg < g; ++gg) before += __popc(ref_word(bitmap, bpr, row, nt * 16 + 4 * gg));
      word = ref_word(bitmap, bpr, row, nt * 16 + 4 * g);
    }
    if (lane == 0) bits[g * kTileK + k] = word;
    if ((word >> lane) & 1u) {
      const uint32_t r = __popc(word & lt);
      const uint32_t ridx = rowtile_off[row * n_nt + nt] + before + r;
      const float v = values_dtype == kF32 ? static_cast<const float*>(values)[ridx]
                                           : __bfloat162float(static_cast<const __nv_bfloat16*>(values)[ridx]);
      if (value_dtype == kBF16)
        reinterpret_cast<__nv_bfloat16*>(rec + kValOffset)[off + r] = __float2bfloat16_rn(v);
      else
        reinterpret_cast<float*>(rec + kValOffset)[off + r] = v;
    }
    off += __popc(word);
  }
  if (threadIdx.x < 16) {
    const uint32_t used = kValOffset + nnz * value_bytes(value_dtype);
    const uint32_t end = 16u * (tile_off[t + 1] - tile_off[t]);
    const uint32_t b = used + threadIdx.x;
    if (b < end) rec[b] = 0;
  }
}

static inline void geometry(int64_t rows, int64_t cols, int64_t* n_kt, int64_t* n_nt) {
  *n_kt = (rows + kTileK - 1) / kTileK;
  *n_nt = (cols + kTileN - 1) / kTileN;
}

static int check_dims(int64_t rows, int64_t cols) {
  SALR_CHECK_ARG(rows >= 1 && cols >= 1, SALR_ERR_SHAPE, "invalid dims (%lld, %lld)", (long long)rows,
                 (long long)cols);
  SALR_CHECK_ARG(rows * cols < (int64_t)0xFFFFFFFF, SALR_ERR_SHAPE,
                 "matrix of %lld entries exceeds the 32-bit value index", (long long)(rows * cols));
  return SALR_OK;
}

}  // namespace salr

using namespace salr;


// ------------------------------------------------------------------ TB2 (compute format)
struct Tb2UnitsFn {
  const uint8_t* records;
  const uint32_t* tile_off;
  __device__ uint32_t operator()(int64_t t) const {
    const uint32_t nnz = reinterpret_cast<const uint32_t*>(records + 16ull * tile_off[t])[3];
    return (uint32_t)((kT2Val + 2u * nnz + 15u) / 16u);
  }
};

// grid = n_tiles, block = 128: thread n <-> tile column n (warp q = column group).
__global__ void tb2_write_kernel(const uint8_t* __restrict__ records, const uint32_t* __restrict__ tile_off,
                                 const uint32_t* __restrict__ tile_off2, uint8_t* __restrict__ records2) {
  const int64_t t = blockIdx.x;
  const int q = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint8_t* src = records + 16ull * tile_off[t];
  uint8_t* dst = records2 + 16ull * tile_off2[t];
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(src);
  const uint32_t* bits = hdr + 4 + q * kTileK;
  const uint32_t goff = q ? hdr[q - 1] : 0u;
  const uint32_t lt = lanemask_lt();
  uint64_t m = 0;
  for (int r = 0; r < kTileK; ++r)
    if ((bits[r] >> l) & 1u) m |= 1ull << r;
  uint32_t excl[16], boff[16];
  uint32_t run = 0;
  for (int b = 0; b < 16; ++b) {
    const uint32_t c = (uint32_t)__popcll((m >> (4 * b)) & 0xFull);
    uint32_t incl = c;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (l >= d) incl += y;
    }
    excl[b] = incl - c;
    boff[b] = run;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(dst)[threadIdx.x] = hdr[threadIdx.x];
  if (l < 16) reinterpret_cast<uint16_t*>(dst + kT2BandOff)[q * 16 + l] = (uint16_t)boff[l];
  reinterpret_cast<uint64_t*>(dst + kT2Mask)[threadIdx.x] = m;
  const uint16_t* sv = reinterpret_cast<const uint16_t*>(src + kValOffset);
  uint16_t* dv = reinterpret_cast<uint16_t*>(dst + kT2Val);
  uint32_t rowpref = 0;
  for (int r = 0; r < kTileK; ++r) {
    const uint32_t w = bits[r];
    if ((w >> l) & 1u) {
      const int b = r >> 2;
      const uint32_t nib = (uint32_t)((m >> (4 * b)) & 0xFull);
      const uint32_t rank = __popc(nib & ((1u << (r & 3)) - 1u));
      dv[goff + boff[b] + excl[b] + rank] = sv[goff + rowpref + __popc(w & lt)];
    }
    rowpref += __popc(w);
  }
  if (threadIdx.x < 16) {
    const uint32_t used = kT2Val + 2u * hdr[3];
    const uint32_t end = 16u * (tile_off2[t + 1] - tile_off2[t]);
    const uint32_t bpos = used + threadIdx.x;
    if (bpos < end) dst[bpos] = 0;
  }
}

// TB records (16-byte units per tile) of a matrix held only in TB2 form.
struct TbFromTb2UnitsFn {
  const uint8_t* records2;
  const uint32_t* tile_off2;
  __device__ uint32_t operator()(int64_t t) const {
    const uint32_t nnz = reinterpret_cast<const uint32_t*>(records2 + 16ull * tile_off2[t])[3];
    return record_units(nnz, 2);
  }
};

// Inverse of tb2_write_kernel (bit-exact): grid = n_tiles, block = 128,
// thread n <-> tile column n.  Rebuilds the bf16 TB record of a tile from its
// TB2 record, so a matrix can keep only the compute format resident.
__global__ void tb_from_tb2_kernel(const uint8_t* __restrict__ records2, const uint32_t* __restrict__ tile_off2,
                                   const uint32_t* __restrict__ tile_off, uint8_t* __restrict__ records) {
  const int64_t t = blockIdx.x;
  const int q = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint8_t* src = records2 + 16ull * tile_off2[t];
  uint8_t* dst = records + 16ull * tile_off[t];
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(src);
  const uint32_t goff = q ? hdr[q - 1] : 0u;
  const uint64_t m = reinterpret_cast<const uint64_t*>(src + kT2Mask)[threadIdx.x];
  const uint16_t* boff = reinterpret_cast<const uint16_t*>(src + kT2BandOff) + q * 16;
  const uint32_t lt = lanemask_lt();
  uint32_t excl[16];
  for (int b = 0; b < 16; ++b) {
    const uint32_t c = (uint32_t)__popcll((m >> (4 * b)) & 0xFull);
    uint32_t incl = c;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (l >= d) incl += y;
    }
    excl[b] = incl - c;
  }
  if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(dst)[threadIdx.x] = hdr[threadIdx.x];
  uint32_t* bits = reinterpret_cast<uint32_t*>(dst + kHdrBytes) + q * kTileK;
  const uint16_t* sv = reinterpret_cast<const uint16_t*>(src + kT2Val);
  uint16_t* dv = reinterpret_cast<uint16_t*>(dst + kValOffset);
  uint32_t rowpref = 0;
  for (int r = 0; r < kTileK; ++r) {
    const uint32_t w = __ballot_sync(0xffffffffu, (uint32_t)(m >> r) & 1u);
    if (l == 0) bits[r] = w;
    if ((w >> l) & 1u) {
      const int b = r >> 2;
      const uint32_t nib = (uint32_t)((m >> (4 * b)) & 0xFull);
      const uint32_t rank = __popc(nib & ((1u << (r & 3)) - 1u));
      dv[goff + rowpref + __popc(w & lt)] = sv[goff + boff[b] + excl[b] + rank];
    }
    rowpref += __popc(w);
  }
  if (threadIdx.x < 16) {
    const uint32_t used = kValOffset + 2u * hdr[3];
    const uint32_t end = 16u * (tile_off[t + 1] - tile_off[t]);
    const uint32_t bpos = used + threadIdx.x;
    if (bpos < end) dst[bpos] = 0;
  }
}

// ------------------------------------------------------------------ NM24
// NM24 records (salr_format.cuh) from a dense bf16 matrix: grid = n_tiles,
// block = 512, thread (band b, 4-column group g).  Groups with more than 2
// nonzeros are counted in *bad (the matrix is not 2:4 along its columns).
// Nonzero = not +-0, as the reference encoder (bitmap.py:150-165).
__global__ void __launch_bounds__(512) nm24_write_kernel(const uint16_t* __restrict__ dense, int64_t rows,
                                                         int64_t cols, int64_t ld, int64_t n_kt,
                                                         uint8_t* __restrict__ out, uint32_t* bad) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int b = threadIdx.x >> 5, g = threadIdx.x & 31;
  const int64_t c0 = nt * kTileN + 4 * g;
  uint32_t w[4];
  uint32_t masks = 0, over = 0;
  for (int r = 0; r < 4; ++r) {
    const int64_t row = kt * kTileK + 4 * b + r;
    uint32_t m = 0, v0 = 0, v1 = 0, n = 0;
    for (int c = 0; c < 4; ++c) {
      const uint32_t bits = (row < rows && c0 + c < cols) ? dense[row * ld + c0 + c] : 0u;
      if (bits & 0x7FFFu) {
        m |= 1u << c;
        if (n == 0) v0 = bits;
        else if (n == 1) v1 = bits;
        ++n;
      }
    }
    over += n > 2;
    w[r] = v0 | v1 << 16;
    masks |= m << (4 * r);
  }
  uint8_t* rec = out + (size_t)t * kNmRecBytes;
  *reinterpret_cast<uint4*>(rec + 16 * (32 * b + g)) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint16_t*>(rec + kNmValBytes + 16 * (32 * (b >> 3) + g) + 4 * ((b & 7) >> 1) + 2 * (b & 1)) =
      (uint16_t)masks;
  if (over) atomicAdd(bad, over);
}

// Dense bf16 matrix (ld) from NM24 records; same thread mapping.
__global__ void __launch_bounds__(512) nm24_decode_kernel(const uint8_t* __restrict__ records, int64_t rows,
                                                          int64_t cols, int64_t n_kt, uint16_t* __restrict__ dense,
                                                          int64_t ld) {
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const int b = threadIdx.x >> 5, g = threadIdx.x & 31;
  const int64_t c0 = nt * kTileN + 4 * g;
  const uint8_t* rec = records + (size_t)t * kNmRecBytes;
  const uint4 wv = *reinterpret_cast<const uint4*>(rec + 16 * (32 * b + g));
  const uint32_t w[4] = {wv.x, wv.y, wv.z, wv.w};
  const uint32_t masks = *reinterpret_cast<const uint16_t*>(rec + kNmValBytes + 16 * (32 * (b >> 3) + g) +
                                                             4 * ((b & 7) >> 1) + 2 * (b & 1));
  for (int r = 0; r < 4; ++r) {
    const int64_t row = kt * kTileK + 4 * b + r;
    if (row >= rows) break;
    const uint32_t m = (masks >> (4 * r)) & 0xFu;
    uint32_t n = 0;
    for (int c = 0; c < 4; ++c) {
      uint32_t v = 0;
      if ((m >> c) & 1u) {
        v = n == 0 ? (w[r] & 0xFFFFu) : n == 1 ? (w[r] >> 16) : 0u;
        ++n;
      }
      if (c0 + c < cols) dense[row * ld + c0 + c] = (uint16_t)v;
    }
  }
}

// Dense bf16 matrix (leading dim ld) straight from TB2 records: grid =
// n_tiles, block = 128 (thread n <-> tile column n, warp q = column group),
// the record staged in shared memory; row r of the tile is one coalesced
// 256-byte store across the block.  (Prefill-size products decode each
// weight once per call into a dense scratch for a tensor-core GEMM.)
__global__ void __launch_bounds__(128) tb2_dense_kernel(const uint8_t* __restrict__ records2,
                                                        const uint32_t* __restrict__ tile_off2, int64_t rows,
                                                        int64_t cols, int64_t n_kt, uint16_t* __restrict__ dense,
                                                        int64_t ld) {
  extern __shared__ __align__(16) uint8_t rec[];
  const int64_t t = blockIdx.x;
  const int64_t nt = t / n_kt, kt = t % n_kt;
  const uint32_t o0 = tile_off2[t], o1 = tile_off2[t + 1];
  const uint4* src = reinterpret_cast<const uint4*>(records2 + 16ull * o0);
  for (uint32_t i = threadIdx.x; i < o1 - o0; i += blockDim.x) reinterpret_cast<uint4*>(rec)[i] = src[i];
  __syncthreads();
  const int n = threadIdx.x, q = n >> 5, l = n & 31;
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec);
  const uint16_t* boff = reinterpret_cast<const uint16_t*>(rec + kT2BandOff) + q * 16;
  const uint64_t m = reinterpret_cast<const uint64_t*>(rec + kT2Mask)[n];
  const uint16_t* vals = reinterpret_cast<const uint16_t*>(rec + kT2Val) + (q ? hdr[q - 1] : 0u);
  const int64_t col = nt * kTileN + n;
  // interior tiles (the common case) skip the per-element bounds checks;
  // one row pointer walks down the column
  const int64_t row0 = kt * kTileK;
  const bool full = row0 + kTileK <= rows && nt * kTileN + kTileN <= cols;
  const int vrows = full ? kTileK : (col < cols ? (int)(rows - row0 < kTileK ? rows - row0 : kTileK) : 0);
  uint16_t* p = dense + row0 * ld + col;
  // the 16 band counts as bytes of 4 words (SWAR nibble popcount), one
  // byte-lane warp scan per word (counts <= 4, sums <= 128)
  uint64_t x = m - ((m >> 1) & 0x5555555555555555ull);
  x = (x & 0x3333333333333333ull) + ((x >> 2) & 0x3333333333333333ull);
  uint32_t cw[4], ew[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t v = (uint32_t)(x >> (16 * w)) & 0xFFFFu;
    cw[w] = (v & 0xFu) | ((v & 0xF0u) << 4) | ((v & 0xF00u) << 8) | ((v & 0xF000u) << 12);
    ew[w] = cw[w];
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ew[w], d);
      if (l >= d) ew[w] += y;
    }
  }
#pragma unroll
  for (int w = 0; w < 4; ++w) ew[w] -= cw[w];
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const uint32_t nib = (uint32_t)((m >> (4 * b)) & 0xFull);
    const uint16_t* vp = vals + boff[b] + ((ew[b >> 2] >> (8 * (b & 3))) & 0xFFu);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint16_t v = 0;
      if ((nib >> i) & 1u) v = *vp++;
      if (4 * b + i < vrows) *p = v;
      p += ld;
    }
  }
}

extern "C" {

int salr_version(void) { return 1; }

const char* salr_last_error(void) { return g_err; }

int salr_tb_geometry(int64_t rows, int64_t cols, int64_t* n_kt, int64_t* n_nt, int64_t* n_tiles) {
  if (int rc = check_dims(rows, cols)) return rc;
  geometry(rows, cols, n_kt, n_nt);
  *n_tiles = *n_kt * *n_nt;
  return SALR_OK;
}

int salr_encode_count(const void* dense, int in_dtype, int64_t rows, int64_t cols, int64_t ld,
                      int value_dtype, uint32_t* tile_cnt, uint32_t* tile_off, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(in_dtype == kF32 || in_dtype == kBF16 || in_dtype == kF64, SALR_ERR_DOMAIN,
                 "unsupported input dtype %d", in_dtype);
  SALR_CHECK_ARG(value_dtype == kF32 || value_dtype == kBF16, SALR_ERR_FORMAT,
                 "unsupported value dtype %d", value_dtype);
  SALR_CHECK_ARG(ld >= cols, SALR_ERR_SHAPE, "leading dim %lld < cols %lld", (long long)ld, (long long)cols);
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  const int64_t n_tiles = n_kt * n_nt;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  encode_count_kernel<<<(unsigned)n_tiles, 128, 0, s>>>(dense, in_dtype, rows, cols, ld, n_kt, tile_cnt);
  SALR_LAUNCH_CHECK();
  scan1_kernel<<<1, 1024, 0, s>>>(TileUnitsFn{tile_cnt, value_bytes(value_dtype)}, n_tiles, tile_off);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_encode_write(const void* dense, int in_dtype, int64_t rows, int64_t cols, int64_t ld,
                      int value_dtype, const uint32_t* tile_cnt, const uint32_t* tile_off,
                      uint8_t* records, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(value_dtype == kF32 || value_dtype == kBF16, SALR_ERR_FORMAT,
                 "unsupported value dtype %d", value_dtype);
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  encode_write_kernel<<<(unsigned)(n_kt * n_nt), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      dense, in_dtype, rows, cols, ld, n_kt, value_dtype, tile_cnt, tile_off, records);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_decode(const uint8_t* records, const uint32_t* tile_off, int value_dtype, int64_t rows,
                int64_t cols, int64_t r0, int64_t r1, int64_t c0, int64_t c1, void* out, int out_dtype,
                int64_t ld_out, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(0 <= r0 && r0 <= r1 && r1 <= rows && 0 <= c0 && c0 <= c1 && c1 <= cols, SALR_ERR_BOUNDS,
                 "window rows [%lld,%lld) cols [%lld,%lld) outside (%lld, %lld)", (long long)r0,
                 (long long)r1, (long long)c0, (long long)c1, (long long)rows, (long long)cols);
  SALR_CHECK_ARG(out_dtype == kF32 || out_dtype == kBF16 || out_dtype == kF64, SALR_ERR_DOMAIN,
                 "unsupported output dtype %d", out_dtype);
  if (r1 == r0 || c1 == c0) return SALR_OK;
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  const int64_t kt0 = r0 / kTileK, kt1 = (r1 + kTileK - 1) / kTileK;
  const int64_t nt0 = c0 / kTileN, nt1 = (c1 + kTileN - 1) / kTileN;
  const int64_t span_k = kt1 - kt0, nblocks = span_k * (nt1 - nt0);
  decode_kernel<<<(unsigned)nblocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      records, tile_off, value_dtype, n_kt, r0, r1, c0, c1, kt0, nt0, span_k, out, out_dtype, ld_out);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_tb_nnz(const uint8_t* records, const uint32_t* tile_off, int64_t n_tiles,
                unsigned long long* nnz_dev, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SALR_CUDA_TRY(cudaMemsetAsync(nnz_dev, 0, sizeof(unsigned long long), s));
  const int blocks = (int)std::min<int64_t>(148 * 4, (n_tiles + 255) / 256 + 1);
  tb_nnz_kernel<<<blocks, 256, 0, s>>>(records, tile_off, n_tiles, nnz_dev);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_to_reference(const uint8_t* records, const uint32_t* tile_off, int value_dtype, int64_t rows,
                      int64_t cols, uint32_t* rowtile_off, uint8_t* bitmap_out, void* values_out,
                      int values_dtype, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(values_dtype == kF32 || values_dtype == kBF16, SALR_ERR_DOMAIN,
                 "unsupported values dtype %d", values_dtype);
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  const int64_t n_tiles = n_kt * n_nt;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // rowtile counts land in rowtile_off[0 .. rows*n_nt) then are scanned in place
  // (the single-block scan reads each item before any later write to it).
  tb_rowtile_count_kernel<<<(unsigned)n_tiles, 64, 0, s>>>(records, tile_off, rows, n_kt, n_nt, rowtile_off);
  SALR_LAUNCH_CHECK();
  scan1_kernel<<<1, 1024, 0, s>>>(ArrayFn{rowtile_off}, rows * n_nt, rowtile_off);
  SALR_LAUNCH_CHECK();
  tb_to_reference_kernel<<<(unsigned)n_tiles, 128, 0, s>>>(records, tile_off, value_dtype, rows, cols, n_kt,
                                                           n_nt, rowtile_off, bitmap_out, values_out,
                                                           values_dtype);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_from_reference_count(const uint8_t* bitmap, int64_t rows, int64_t cols, int value_dtype,
                              uint32_t* rowtile_off, uint32_t* tile_cnt, uint32_t* tile_off, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(value_dtype == kF32 || value_dtype == kBF16, SALR_ERR_FORMAT,
                 "unsupported value dtype %d", value_dtype);
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  const int64_t n_tiles = n_kt * n_nt;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nrt = rows * n_nt;
  ref_rowtile_count_kernel<<<(unsigned)((nrt + 255) / 256), 256, 0, s>>>(bitmap, rows, cols, n_nt, rowtile_off);
  SALR_LAUNCH_CHECK();
  scan1_kernel<<<1, 1024, 0, s>>>(ArrayFn{rowtile_off}, nrt, rowtile_off);
  SALR_LAUNCH_CHECK();
  ref_tile_count_kernel<<<(unsigned)((n_tiles * kGroups + 255) / 256), 256, 0, s>>>(bitmap, rows, cols, n_kt,
                                                                                   n_tiles, tile_cnt);
  SALR_LAUNCH_CHECK();
  scan1_kernel<<<1, 1024, 0, s>>>(TileUnitsFn{tile_cnt, value_bytes(value_dtype)}, n_tiles, tile_off);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_from_reference_write(const uint8_t* bitmap, const void* values, int values_dtype, int64_t rows,
                              int64_t cols, int value_dtype, const uint32_t* rowtile_off,
                              const uint32_t* tile_cnt, const uint32_t* tile_off, uint8_t* records,
                              void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(values_dtype == kF32 || values_dtype == kBF16, SALR_ERR_DOMAIN,
                 "unsupported values dtype %d", values_dtype);
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  ref_to_tb_kernel<<<(unsigned)(n_kt * n_nt), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      bitmap, values, values_dtype, rows, cols, n_kt, n_nt, value_dtype, rowtile_off, tile_cnt, tile_off,
      records);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}


int salr_tb2_count(const uint8_t* records, const uint32_t* tile_off, int64_t rows, int64_t cols,
                   uint32_t* tile_off2, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  scan1_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(Tb2UnitsFn{records, tile_off}, n_kt * n_nt,
                                                                  tile_off2);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_tb2_write(const uint8_t* records, const uint32_t* tile_off, int64_t rows, int64_t cols,
                   const uint32_t* tile_off2, uint8_t* records2, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  tb2_write_kernel<<<(unsigned)(n_kt * n_nt), 128, 0, static_cast<cudaStream_t>(stream)>>>(records, tile_off,
                                                                                           tile_off2, records2);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_tb_from_tb2_count(const uint8_t* records2, const uint32_t* tile_off2, int64_t rows, int64_t cols,
                          uint32_t* tile_off, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  scan1_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(TbFromTb2UnitsFn{records2, tile_off2},
                                                                  n_kt * n_nt, tile_off);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_tb_from_tb2_write(const uint8_t* records2, const uint32_t* tile_off2, int64_t rows, int64_t cols,
                          const uint32_t* tile_off, uint8_t* records, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  tb_from_tb2_kernel<<<(unsigned)(n_kt * n_nt), 128, 0, static_cast<cudaStream_t>(stream)>>>(records2, tile_off2,
                                                                                             tile_off, records);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_nm24_write(const void* dense_bf16, int64_t rows, int64_t cols, int64_t ld, uint8_t* records,
                    uint32_t* bad_groups, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(ld >= cols, SALR_ERR_SHAPE, "ld < cols");
  SALR_CHECK_ARG(dense_bf16 && records && bad_groups, SALR_ERR_CONFIG, "null pointer");
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  nm24_write_kernel<<<(unsigned)(n_kt * n_nt), 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(dense_bf16), rows, cols, ld, n_kt, records, bad_groups);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_nm24_decode(const uint8_t* records, int64_t rows, int64_t cols, void* dense_bf16, int64_t ld,
                     void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(ld >= cols, SALR_ERR_SHAPE, "ld < cols");
  SALR_CHECK_ARG(dense_bf16 && records, SALR_ERR_CONFIG, "null pointer");
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  nm24_decode_kernel<<<(unsigned)(n_kt * n_nt), 512, 0, static_cast<cudaStream_t>(stream)>>>(
      records, rows, cols, n_kt, static_cast<uint16_t*>(dense_bf16), ld);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_tb2_decode(const uint8_t* records2, const uint32_t* tile_off2, int64_t rows, int64_t cols,
                    void* dense_bf16, int64_t ld, void* stream) {
  if (int rc = check_dims(rows, cols)) return rc;
  SALR_CHECK_ARG(ld >= cols, SALR_ERR_SHAPE, "ld < cols");
  SALR_CHECK_ARG(records2 && tile_off2 && dense_bf16, SALR_ERR_CONFIG, "null pointer");
  int64_t n_kt, n_nt;
  geometry(rows, cols, &n_kt, &n_nt);
  // one 17.6 KB record slot per 128-thread block: ask for the shared-memory
  // carve-out that lets ~12 blocks share an SM (the default may leave 1-2)
  static bool carve[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !carve[dev]) {
    cudaFuncSetAttribute(tb2_dense_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    carve[dev] = true;
  }
  tb2_dense_kernel<<<(unsigned)(n_kt * n_nt), 128, kMaxRecordBytesT2 + 16, static_cast<cudaStream_t>(stream)>>>(
      records2, tile_off2, rows, cols, n_kt, static_cast<uint16_t*>(dense_bf16), ld);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

}  // extern "C"
