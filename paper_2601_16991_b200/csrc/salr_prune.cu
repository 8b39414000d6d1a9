// Exact magnitude-prune masks on the device (reference pkg/src/salr/prune.py:
// build_mask 224-255, _largest_mask_flat 215-221).
//
// Global methods keep exactly `keep` = kept_count(p, rows*cols) entries: the
// largest scores, ties broken toward the lower row-major index -- the stable
// argsort of the reference.  Here: an MSB-first radix select (8-bit digits)
// finds the keep-th largest score T and how many entries equal to T survive;
// a block-ordered scan then keeps the lowest-index ties.  All state lives in
// the caller's workspace; every step is stream-ordered (no host sync).
//
// N:M keeps the n largest |w| of every contiguous group of m columns, ties
// toward the lower column offset (prune.py:238-248).
//
// Scores are non-negative (|w|, |w + delta|), so their IEEE bit patterns order
// like the values; float32 scores widen to the float64 order exactly.

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "salr_status.cuh"

namespace salr {

constexpr int kPruneThreads = 256;
constexpr int kPruneItems = 8;  // elements per thread in the mask passes

struct SelectState {
  unsigned long long prefix;       // high digits of T found so far
  unsigned long long prefix_mask;  // which bits of prefix are fixed
  unsigned long long k_rem;        // still to select among prefix matches
  unsigned long long n_keep;       // total to keep
};

__device__ __forceinline__ unsigned long long score_key(const void* s, int f64, int64_t i) {
  if (f64) {
    const unsigned long long b = static_cast<const unsigned long long*>(s)[i];
    return b & 0x7FFFFFFFFFFFFFFFull;
  }
  // float32 -> float64 bit pattern order: widen exactly
  const double d = (double)fabsf(static_cast<const float*>(s)[i]);
  return (unsigned long long)__double_as_longlong(d);
}

__global__ void select_init_kernel(SelectState* st, uint32_t* hist, unsigned long long keep) {
  st->prefix = 0ull;
  st->prefix_mask = 0ull;
  st->k_rem = keep;
  st->n_keep = keep;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
}

__global__ void __launch_bounds__(kPruneThreads) select_hist_kernel(const void* s, int f64, int64_t n, int shift,
                                                                    const SelectState* st, uint32_t* hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const unsigned long long pre = st->prefix, pm = st->prefix_mask;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = score_key(s, f64, i);
    if ((k & pm) == pre) atomicAdd(&h[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// One thread: pick the digit of T at `shift` (largest digits first).
__global__ void select_digit_kernel(SelectState* st, uint32_t* hist, int shift) {
  if (threadIdx.x != 0) return;
  unsigned long long k = st->k_rem, above = 0;
  int d = 255;
  for (; d > 0; --d) {
    if (above + hist[d] >= k) break;
    above += hist[d];
  }
  st->k_rem = k - above;
  st->prefix |= (unsigned long long)d << shift;
  st->prefix_mask |= 255ull << shift;
  for (int i = 0; i < 256; ++i) hist[i] = 0u;
}

// Pass A: entries equal to T per block (block = kPruneThreads * kPruneItems
// consecutive elements).
__global__ void __launch_bounds__(kPruneThreads) tie_count_kernel(const void* s, int f64, int64_t n,
                                                                  const SelectState* st, uint32_t* block_ties) {
  __shared__ uint32_t cnt;
  if (threadIdx.x == 0) cnt = 0u;
  __syncthreads();
  const unsigned long long T = st->prefix;
  const int64_t base = (int64_t)blockIdx.x * kPruneThreads * kPruneItems;
  uint32_t c = 0;
  for (int j = 0; j < kPruneItems; ++j) {
    const int64_t i = base + (int64_t)j * kPruneThreads + threadIdx.x;
    if (i < n && score_key(s, f64, i) == T) ++c;
  }
  if (c) atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) block_ties[blockIdx.x] = cnt;
}

// Exclusive scan of the per-block tie counts (one block, sequential chunks).
__global__ void __launch_bounds__(1024) tie_scan_kernel(uint32_t* block_ties, int64_t nb) {
  __shared__ uint32_t carry;
  __shared__ uint32_t warp_sum[32];
  if (threadIdx.x == 0) carry = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t c0 = 0; c0 < nb; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    const uint32_t v = i < nb ? block_ties[i] : 0u;
    uint32_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t w = warp_sum[lane];
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      warp_sum[lane] = w;
    }
    __syncthreads();
    const uint32_t incl = x + (wid ? warp_sum[wid - 1] : 0u) + carry;
    if (i < nb) block_ties[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
}

// Pass B: keep > T, and the first k_rem entries == T in row-major order.
__global__ void __launch_bounds__(kPruneThreads) mask_write_kernel(const void* s, int f64, int64_t n,
                                                                   const SelectState* st,
                                                                   const uint32_t* block_ties, uint8_t* mask) {
  __shared__ uint32_t warp_tot[kPruneThreads / 32];
  const unsigned long long T = st->prefix, k_rem = st->k_rem;
  const bool none = st->n_keep == 0ull;
  const int64_t base = (int64_t)blockIdx.x * kPruneThreads * kPruneItems;
  uint32_t run = block_ties[blockIdx.x];  // ties before this block
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = 0; j < kPruneItems; ++j) {
    const int64_t i = base + (int64_t)j * kPruneThreads + threadIdx.x;
    const unsigned long long k = i < n ? score_key(s, f64, i) : 0ull;
    const bool tie = i < n && k == T;
    const uint32_t bal = __ballot_sync(0xffffffffu, tie);
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    uint32_t before = run + __popc(bal & ((1u << lane) - 1u));
    for (int w = 0; w < wid; ++w) before += warp_tot[w];
    uint32_t chunk = 0;
    for (int w = 0; w < kPruneThreads / 32; ++w) chunk += warp_tot[w];
    if (i < n) mask[i] = (uint8_t)(!none && (k > T || (tie && (unsigned long long)before < k_rem)));
    run += chunk;
    __syncthreads();
  }
}

// N:M: one thread per (row, group); keep the n largest of m scores, ties to
// the lower offset: element j is kept iff fewer than n entries rank above it.
__global__ void nm_mask_kernel(const void* s, int f64, int64_t rows, int64_t cols, int nn, int mm, uint8_t* mask) {
  const int64_t groups = rows * (cols / mm);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = g * mm;  // groups are contiguous in row-major order
    for (int j = 0; j < mm; ++j) {
      const unsigned long long kj = score_key(s, f64, base + j);
      int above = 0;
      for (int t = 0; t < mm; ++t) {
        const unsigned long long kt = score_key(s, f64, base + t);
        above += (kt > kj) || (kt == kj && t < j);
      }
      mask[base + j] = (uint8_t)(above < nn);
    }
  }
}

}  // namespace salr

using namespace salr;

extern "C" {

size_t salr_topk_mask_workspace_bytes(int64_t n) {
  const int64_t nb = (n + kPruneThreads * kPruneItems - 1) / (kPruneThreads * kPruneItems);
  return 256 + 256 * 4 + (size_t)(nb + 1) * 4;
}

int salr_topk_mask(const void* scores, int dtype, int64_t n, int64_t keep, uint8_t* mask, void* workspace,
                   size_t workspace_bytes, void* stream) {
  SALR_CHECK_ARG(n >= 1, SALR_ERR_SHAPE, "empty score array");
  SALR_CHECK_ARG(dtype == 0 || dtype == 2, SALR_ERR_DOMAIN, "scores must be float32 (0) or float64 (2)");
  SALR_CHECK_ARG(keep >= 0 && keep <= n, SALR_ERR_DOMAIN, "keep %lld outside [0, %lld]", (long long)keep,
                 (long long)n);
  SALR_CHECK_ARG(workspace_bytes >= salr_topk_mask_workspace_bytes(n), SALR_ERR_CONFIG, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  SelectState* st = reinterpret_cast<SelectState*>(ws);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + 256);
  uint32_t* block_ties = reinterpret_cast<uint32_t*>(ws + 256 + 256 * 4);
  const int f64 = dtype == 2;
  const int64_t nb = (n + kPruneThreads * kPruneItems - 1) / (kPruneThreads * kPruneItems);
  select_init_kernel<<<1, 256, 0, s>>>(st, hist, (unsigned long long)keep);
  SALR_LAUNCH_CHECK();
  if (keep > 0) {
    const int top = 56;  // keys have the sign bit clear: 63 value bits, top digit at bits 56-63
    const int64_t grid = std::min<int64_t>((n + kPruneThreads - 1) / kPruneThreads, 148 * 8);
    for (int shift = top; shift >= 0; shift -= 8) {
      select_hist_kernel<<<(unsigned)grid, kPruneThreads, 0, s>>>(scores, f64, n, shift, st, hist);
      select_digit_kernel<<<1, 32, 0, s>>>(st, hist, shift);
    }
    SALR_LAUNCH_CHECK();
  }
  tie_count_kernel<<<(unsigned)nb, kPruneThreads, 0, s>>>(scores, f64, n, st, block_ties);
  tie_scan_kernel<<<1, 1024, 0, s>>>(block_ties, nb);
  mask_write_kernel<<<(unsigned)nb, kPruneThreads, 0, s>>>(scores, f64, n, st, block_ties, mask);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

int salr_nm_mask(const void* scores, int dtype, int64_t rows, int64_t cols, int n_keep, int m_group, uint8_t* mask,
                 void* stream) {
  SALR_CHECK_ARG(rows >= 1 && cols >= 1, SALR_ERR_SHAPE, "invalid dims (%lld, %lld)", (long long)rows,
                 (long long)cols);
  SALR_CHECK_ARG(dtype == 0 || dtype == 2, SALR_ERR_DOMAIN, "scores must be float32 (0) or float64 (2)");
  SALR_CHECK_ARG(0 < n_keep && n_keep < m_group && m_group <= 64, SALR_ERR_CONFIG, "nm requires 0 < n < m <= 64");
  SALR_CHECK_ARG(cols % m_group == 0, SALR_ERR_CONFIG, "group size m=%d must divide cols=%lld", m_group,
                 (long long)cols);
  const int64_t groups = rows * (cols / m_group);
  const int64_t grid = std::min<int64_t>((groups + 255) / 256, 148 * 16);
  nm_mask_kernel<<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(scores, dtype == 2, rows, cols,
                                                                                n_keep, m_group, mask);
  SALR_LAUNCH_CHECK();
  return SALR_OK;
}

}  // extern "C"
