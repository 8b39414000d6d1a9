// Micro-benchmark of the TB2 tile decoder in isolation: records resident in
// shared memory, 16 decoder warps (4 groups x 4 column blocks) expanding
// 64x128 tiles into the TMEM A operand with tcgen05.st, no MMA, no TMA.
// Reports SM cycles per decoded tile (all 148 SMs busy) and checks the TMEM
// contents of one decode against the host expansion.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -o tools/ubench/ubench_decode tools/ubench/ubench_decode.cu -lcuda
//   tools/ubench/ubench_decode [p=0.5]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2601_16991_b200/csrc/salr_format.cuh"
#include "../../paper_2601_16991_b200/csrc/salr_ptx.cuh"
using namespace salr;

constexpr int kR = 8;             // records resident per CTA
constexpr uint32_t kSlot = 10240; // bytes per record slot
constexpr int kDecWarps = 16;
#ifndef MMA_PROBE
#define MMA_PROBE 1
#endif
constexpr bool kMmaProbe = MMA_PROBE;

__host__ __device__ constexpr uint32_t nib_sel(uint32_t x) {
  return x == 0 ? 0x3232u : x == 1 ? 0x3210u : x == 2 ? 0x1032u : 0x5410u;
}
__host__ __device__ constexpr uint64_t nib_lut_entry(uint32_t n) {
  return (uint64_t)(nib_sel(n & 3u) | ((2u * ((n & 1u) + ((n >> 1) & 1u))) << 16)) |
         ((uint64_t)nib_sel(n >> 2) << 32);
}

// ---------------------------------------------------------------- V0: round-2 kernel decoder
__device__ __forceinline__ void decode_v0(const uint8_t* rec, uint32_t taddr, int q, uint32_t lane,
                                          const uint64_t* s_lut, const uint8_t* smem_raw) {
  constexpr int BPW = 16;
  const uint2 mw = *reinterpret_cast<const uint2*>(rec + kT2Mask + 8 * (32 * q + lane));
  const uint32_t goff = q ? reinterpret_cast<const uint32_t*>(rec)[q - 1] : 0u;
  const uint4 bo0 = *reinterpret_cast<const uint4*>(rec + kT2BandOff + 32 * q);
  const uint4 bo1 = *reinterpret_cast<const uint4*>(rec + kT2BandOff + 32 * q + 16);
  const uint32_t bo[8] = {bo0.x, bo0.y, bo0.z, bo0.w, bo1.x, bo1.y, bo1.z, bo1.w};
  uint32_t nl = mw.x - ((mw.x >> 1) & 0x55555555u);
  nl = (nl & 0x33333333u) + ((nl >> 2) & 0x33333333u);
  uint32_t nh = mw.y - ((mw.y >> 1) & 0x55555555u);
  nh = (nh & 0x33333333u) + ((nh >> 2) & 0x33333333u);
  const uint32_t c[4] = {nl & 0x0F0F0F0Fu, (nl >> 4) & 0x0F0F0F0Fu, nh & 0x0F0F0F0Fu, (nh >> 4) & 0x0F0F0F0Fu};
  uint32_t e[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = __shfl_up_sync(0xffffffffu, e[j], d);
    if ((int)lane >= d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] += t[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] -= c[j];
  const uint32_t vbase = smem_u32(rec) + kT2Val + 2u * goff;
  const uint32_t smem_base_u32 = smem_u32(smem_raw);
#pragma unroll
  for (int c4 = 0; c4 < BPW / 4; ++c4) {
    uint32_t packed[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int b = 4 * c4 + i;
      const uint32_t ev = e[(b >= 8 ? 2 : 0) + (b & 1)];
      const uint32_t ex = prmt(ev, 0u, 0x4440u + (uint32_t)((b & 7) >> 1));
      const uint32_t bov = prmt(bo[b >> 1], 0u, (b & 1) ? 0x4432u : 0x4410u);
      const uint32_t r = vbase + 2u * (bov + ex);
      const uint32_t word = b < 8 ? mw.x : mw.y;
      const int sh = 4 * (b & 7);
      const uint32_t nib8 = sh >= 3 ? ((word >> (sh - 3)) & 0x78u) : ((word << 3) & 0x78u);
      const uint2 ent = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(s_lut) + nib8);
      const uint32_t e0 = ent.x, e1 = ent.y;
      const uint8_t* rp = smem_raw + (r - smem_base_u32);
      const uint8_t* rp2 = rp + (e0 >> 16);
      const uint32_t a0 = *reinterpret_cast<const uint16_t*>(rp);
      const uint32_t a1 = *reinterpret_cast<const uint16_t*>(rp + 2);
      const uint32_t b0 = *reinterpret_cast<const uint16_t*>(rp2);
      const uint32_t b1 = *reinterpret_cast<const uint16_t*>(rp2 + 2);
      packed[2 * i] = prmt(a0, a1, e0);
      packed[2 * i + 1] = prmt(b0, b1, e1);
    }
    SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
  }
  tc_wait_st();
}

// ---------------------------------------------------------------- V1: lean band decoder
__device__ __forceinline__ uint32_t lds_u16a(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lea_hi16(uint32_t x, uint32_t base) {  // base + (x >> 16)
  return base + (x >> 16);
}

// lut_base: shared address of the 16-entry nibble table, 128-byte aligned.
template <int kVar>
__device__ __forceinline__ void decode_v1(uint32_t rec, uint32_t taddr, int q, uint32_t lane, uint32_t lut_base) {
  const uint2 mw = lds_v2(rec + kT2Mask + 8 * (32 * q + lane));
  // band counts as bytes: c0 bands 0,2,4,6; c1 1,3,5,7; c2 8..14 even; c3 9..15 odd
  uint32_t nl = mw.x - ((mw.x >> 1) & 0x55555555u);
  nl = (nl & 0x33333333u) + ((nl >> 2) & 0x33333333u);
  uint32_t nh = mw.y - ((mw.y >> 1) & 0x55555555u);
  nh = (nh & 0x33333333u) + ((nh >> 2) & 0x33333333u);
  const uint32_t c[4] = {nl & 0x0F0F0F0Fu, (nl >> 4) & 0x0F0F0F0Fu, nh & 0x0F0F0F0Fu, (nh >> 4) & 0x0F0F0F0Fu};
  uint32_t e[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = __shfl_up_sync(0xffffffffu, e[j], d);
    if ((int)lane >= d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] += t[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] -= c[j];
  // band offsets (u16 pairs, warp-uniform) + group base
  uint32_t hdr_q;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hdr_q) : "r"(rec + 4 * (q - 1)));
  const uint32_t vb = rec + kT2Val + 2u * (q ? hdr_q : 0u);
  uint32_t bo[8];
  {
    uint4 b0, b1;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b0.x), "=r"(b0.y), "=r"(b0.z), "=r"(b0.w)
                 : "r"(rec + kT2BandOff + 32 * q));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b1.x), "=r"(b1.y), "=r"(b1.z), "=r"(b1.w)
                 : "r"(rec + kT2BandOff + 32 * q + 16));
    bo[0] = b0.x; bo[1] = b0.y; bo[2] = b0.z; bo[3] = b0.w;
    bo[4] = b1.x; bo[5] = b1.y; bo[6] = b1.z; bo[7] = b1.w;
  }
  const uint32_t m8[2] = {mw.x << 3, mw.y << 3};
  const uint32_t m8h[2] = {mw.x >> 1, mw.y >> 1};  // for nibbles >= 1: (m >> (4b-3))
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    uint32_t packed[8];
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const int b = 4 * c4 + i;  // bands b, b+1 (b even)
      // 16-bit pair (prefix[b], prefix[b+1]): bytes of e[] are < 128 -> sign-replicate gives 0
      const int j = (b & 7) >> 1;
      const uint32_t ea = e[b >= 8 ? 2 : 0], eb = e[b >= 8 ? 3 : 1];
      const uint32_t sel = (uint32_t)j | ((0x8u | j) << 4) | ((4u + j) << 8) | ((0x8u | j) << 12);
      const uint32_t pr = prmt(ea, eb, sel) + bo[b >> 1];  // (e[b] + bo[b]) | (e[b+1] + bo[b+1]) << 16
      const uint32_t ra = vb + 2u * (pr & 0xFFFFu);
      const uint32_t rb = vb + (pr >> 15);  // bit 15 of the low half is 0
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bb = b + h;
        const uint32_t r = h ? rb : ra;
        const int sh = 4 * (bb & 7);
        const uint32_t word = bb < 8 ? mw.x : mw.y;
        const uint32_t nib8 = sh ? ((word >> (sh - 3)) & 0x78u) : ((word << 3) & 0x78u);
        const uint2 ent = lds_v2(lut_base | nib8);
        const uint32_t r2 = lea_hi16(ent.x, r);
        const uint32_t a0 = lds_u16a(r), a1 = lds_u16a(r + 2);
        const uint32_t b0 = lds_u16a(r2), b1 = lds_u16a(r2 + 2);
        packed[2 * (i + h)] = prmt(a0, a1, ent.x);
        packed[2 * (i + h) + 1] = prmt(b0, b1, ent.y);
      }
    }
    SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
  }
  tc_wait_st();
  (void)m8; (void)m8h;
}


// ---------------------------------------------------------------- V2: 3 aligned words per band run
// Window of the band run = halfwords e..e+3, fetched as the three aligned
// words around e (ld.shared.u32) and funnel-shifted into V0 = [h0,h1],
// V1 = [h2,h3].  Row pair 0 takes h0,h1; row pair 1 takes h(c0),h(c0+1)
// (c0 = present rows of pair 0) via a clamped funnel shift; absent rows pick
// zero bytes of RZ in the final byte permute.
__host__ __device__ constexpr uint32_t sel_z(uint32_t x) {  // window [lo,hi] -> rows (x bit0, x bit1), zeros from RZ
  return x == 0 ? 0x4444u : x == 1 ? 0x4410u : x == 2 ? 0x1044u : 0x3210u;
}
__host__ __device__ constexpr uint32_t lut2_entry(uint32_t n) { return sel_z(n & 3u) | (sel_z(n >> 2) << 16); }

__device__ __forceinline__ void decode_v2(uint32_t rec, uint32_t taddr, int q, uint32_t lane, uint32_t lut_base) {
  const uint2 mw = lds_v2(rec + kT2Mask + 8 * (32 * q + lane));
  const uint32_t pl = mw.x - ((mw.x >> 1) & 0x55555555u);  // 2-bit pair counts
  const uint32_t ph = mw.y - ((mw.y >> 1) & 0x55555555u);
  const uint32_t nl = (pl & 0x33333333u) + ((pl >> 2) & 0x33333333u);
  const uint32_t nh = (ph & 0x33333333u) + ((ph >> 2) & 0x33333333u);
  const uint32_t c[4] = {nl & 0x0F0F0F0Fu, (nl >> 4) & 0x0F0F0F0Fu, nh & 0x0F0F0F0Fu, (nh >> 4) & 0x0F0F0F0Fu};
  uint32_t e[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = __shfl_up_sync(0xffffffffu, e[j], d);
    if ((int)lane >= d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] += t[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] -= c[j];
  uint32_t hdr_q = 0;
  if (q) hdr_q = lds_u32(rec + 4 * (q - 1));
  const uint32_t vb = rec + kT2Val + 2u * hdr_q;
  uint32_t bo[8];
  {
    uint4 b0, b1;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b0.x), "=r"(b0.y), "=r"(b0.z), "=r"(b0.w)
                 : "r"(rec + kT2BandOff + 32 * q));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b1.x), "=r"(b1.y), "=r"(b1.z), "=r"(b1.w)
                 : "r"(rec + kT2BandOff + 32 * q + 16));
    bo[0] = b0.x; bo[1] = b0.y; bo[2] = b0.z; bo[3] = b0.w;
    bo[4] = b1.x; bo[5] = b1.y; bo[6] = b1.z; bo[7] = b1.w;
  }
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    uint32_t packed[8];
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const int b = 4 * c4 + i;
      const int j = (b & 7) >> 1;
      const uint32_t ea = e[b >= 8 ? 2 : 0], eb = e[b >= 8 ? 3 : 1];
      const uint32_t sel = (uint32_t)j | ((0x8u | j) << 4) | ((4u + j) << 8) | ((0x8u | j) << 12);
      const uint32_t pr = prmt(ea, eb, sel) + bo[b >> 1];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bb = b + h;
        const uint32_t r = h ? vb + (pr >> 15) : vb + 2u * (pr & 0xFFFFu);
        const uint32_t wa = r & ~3u, amt = r << 3;
        const uint32_t A = lds_u32(wa), B = lds_u32(wa + 4), C = lds_u32(wa + 8);
        const int sh = 4 * (bb & 7);
        const uint32_t word = bb < 8 ? mw.x : mw.y;
        const uint32_t pcw = bb < 8 ? pl : ph;
        const uint32_t nib4 = (sh >= 2 ? (word >> (sh - 2)) : (word << 2)) & 0x3Cu;
        const uint32_t ent = lds_u32(lut_base | nib4);
        const uint32_t c0sh = (sh >= 4 ? (pcw >> (sh - 4)) : (pcw << 4)) & 0x30u;
        const uint32_t V0 = shf_r_wrap(A, B, amt), V1 = shf_r_wrap(B, C, amt);
        const uint32_t Vp = shf_r_clamp(V0, V1, c0sh);
        packed[2 * (i + h)] = prmt(V0, 0u, ent);
        packed[2 * (i + h) + 1] = prmt(Vp, 0u, ent >> 16);
      }
    }
    SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
  }
  tc_wait_st();
}

__device__ __forceinline__ void decode_v3(uint32_t rec, uint32_t taddr, int q, uint32_t lane, uint32_t lut_base) {
  const uint2 mw = lds_v2(rec + kT2Mask + 8 * (32 * q + lane));
  const uint32_t pl = mw.x - ((mw.x >> 1) & 0x55555555u);  // 2-bit pair counts
  const uint32_t ph = mw.y - ((mw.y >> 1) & 0x55555555u);
  const uint32_t nl = (pl & 0x33333333u) + ((pl >> 2) & 0x33333333u);
  const uint32_t nh = (ph & 0x33333333u) + ((ph >> 2) & 0x33333333u);
  const uint32_t c[4] = {nl & 0x0F0F0F0Fu, (nl >> 4) & 0x0F0F0F0Fu, nh & 0x0F0F0F0Fu, (nh >> 4) & 0x0F0F0F0Fu};
  uint32_t e[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = __shfl_up_sync(0xffffffffu, e[j], d);
    if ((int)lane >= d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] += t[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] -= c[j];
  uint32_t hdr_q = 0;
  if (q) hdr_q = lds_u32(rec + 4 * (q - 1));
  const uint32_t vb = rec + kT2Val + 2u * hdr_q;
  uint32_t bo[8];
  {
    uint4 b0, b1;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b0.x), "=r"(b0.y), "=r"(b0.z), "=r"(b0.w)
                 : "r"(rec + kT2BandOff + 32 * q));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b1.x), "=r"(b1.y), "=r"(b1.z), "=r"(b1.w)
                 : "r"(rec + kT2BandOff + 32 * q + 16));
    bo[0] = b0.x; bo[1] = b0.y; bo[2] = b0.z; bo[3] = b0.w;
    bo[4] = b1.x; bo[5] = b1.y; bo[6] = b1.z; bo[7] = b1.w;
  }
  uint32_t bo2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) bo2[k] = bo[k] + bo[k];
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    uint32_t packed[8];
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const int b = 4 * c4 + i;
      const int j = (b & 7) >> 1;
      const uint32_t ea = e[b >= 8 ? 2 : 0], eb = e[b >= 8 ? 3 : 1];
      const uint32_t sel = (uint32_t)j | ((0x8u | j) << 4) | ((4u + j) << 8) | ((0x8u | j) << 12);
      const uint32_t pp = prmt(ea, eb, sel);
      const uint32_t pr2 = pp + pp + bo2[b >> 1];  // byte offsets of bands b, b+1 (16-bit lanes)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bb = b + h;
        const uint32_t wa = vb + (h ? ((pr2 >> 16) & 0xFFFCu) : (pr2 & 0xFFFCu));
        const uint32_t amt = h ? (pr2 >> 13) : (pr2 << 3);
        const uint32_t A = lds_u32(wa), B = lds_u32(wa + 4), C = lds_u32(wa + 8);
        const int sh = 4 * (bb & 7);
        const uint32_t word = bb < 8 ? mw.x : mw.y;
        const uint32_t pcw = bb < 8 ? pl : ph;
        const uint32_t nib4 = (sh >= 2 ? (word >> (sh - 2)) : (word << 2)) & 0x3Cu;
        const uint32_t ent = lds_u32(lut_base | nib4);
        const uint32_t c0sh = (sh >= 4 ? (pcw >> (sh - 4)) : (pcw << 4)) & 0x30u;
        const uint32_t V0 = shf_r_wrap(A, B, amt), V1 = shf_r_wrap(B, C, amt);
        const uint32_t Vp = shf_r_clamp(V0, V1, c0sh);
        packed[2 * (i + h)] = prmt(V0, 0u, ent);
        packed[2 * (i + h) + 1] = prmt(Vp, 0u, ent >> 16);
      }
    }
    SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
  }
  tc_wait_st();
}


// ---------------------------------------------------------------- V4: V0 loads, lean addressing
// 4 zero-extended u16 loads per band + 64-bit nibble entry (sel0 | 2c0 << 16, sel1),
// run addresses from 16-bit pairs of (prefix + band offset) in bytes.
__device__ __forceinline__ void decode_v4(uint32_t rec, uint32_t taddr, int q, uint32_t lane, uint32_t lut_base) {
  const uint2 mw = lds_v2(rec + kT2Mask + 8 * (32 * q + lane));
  uint32_t nl = mw.x - ((mw.x >> 1) & 0x55555555u);
  nl = (nl & 0x33333333u) + ((nl >> 2) & 0x33333333u);
  uint32_t nh = mw.y - ((mw.y >> 1) & 0x55555555u);
  nh = (nh & 0x33333333u) + ((nh >> 2) & 0x33333333u);
  const uint32_t c[4] = {nl & 0x0F0F0F0Fu, (nl >> 4) & 0x0F0F0F0Fu, nh & 0x0F0F0F0Fu, (nh >> 4) & 0x0F0F0F0Fu};
  uint32_t e[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = __shfl_up_sync(0xffffffffu, e[j], d);
    if ((int)lane >= d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] += t[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] -= c[j];
  uint32_t goff = 0;
  if (q) goff = lds_u32(rec + 4 * (q - 1));
  const uint32_t vb = rec + kT2Val + 2u * goff;
  uint4 b0, b1;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b0.x), "=r"(b0.y), "=r"(b0.z), "=r"(b0.w)
               : "r"(rec + kT2BandOff + 32 * q));
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b1.x), "=r"(b1.y), "=r"(b1.z), "=r"(b1.w)
               : "r"(rec + kT2BandOff + 32 * q + 16));
  const uint32_t bo[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    uint32_t packed[8];
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const int b = 4 * c4 + i;
      const int j = (b & 7) >> 1;
      const uint32_t pe = prmt(e[b >= 8 ? 2 : 0], e[b >= 8 ? 3 : 1],
                               (uint32_t)j | ((0x8u | j) << 4) | ((4u + j) << 8) | ((0x8u | j) << 12));
      const uint32_t pr2 = pe + pe + (bo[b >> 1] + bo[b >> 1]);  // byte offsets, 16-bit lanes
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bb = b + h;
        const uint32_t r = h ? vb + (pr2 >> 16) : vb + (pr2 & 0xFFFFu);
        const int sh = 4 * (bb & 7);
        const uint32_t word = bb < 8 ? mw.x : mw.y;
        const uint32_t nib8 = (sh >= 3 ? (word >> (sh - 3)) : (word << 3)) & 0x78u;
        const uint2 ent = lds_v2(lut_base | nib8);
        const uint32_t r2 = r + (ent.x >> 16);
        const uint32_t a0 = lds_u16z(r), a1 = lds_u16z(r + 2);
        const uint32_t c0 = lds_u16z(r2), c1 = lds_u16z(r2 + 2);
        packed[2 * (i + h)] = prmt(a0, a1, ent.x);
        packed[2 * (i + h) + 1] = prmt(c0, c1, ent.y);
      }
    }
    SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
  }
  tc_wait_st();
}

template <int kVar>
__global__ void __launch_bounds__(32 * (kDecWarps + 1), 1)
bench_kernel(const uint8_t* __restrict__ recs, const uint32_t* __restrict__ rec_bytes, int iters,
             long long* __restrict__ cycles, uint32_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(128) uint64_t s_lut[16];
  __shared__ __align__(128) uint32_t s_lut2[16];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kR * (int)kSlot / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(recs)[i];
  if (threadIdx.x < 16) s_lut[threadIdx.x] = nib_lut_entry(threadIdx.x);
  if (threadIdx.x < 16) s_lut2[threadIdx.x] = lut2_entry(threadIdx.x);
  if (warp == 0) tmem_alloc(&tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  __shared__ __align__(8) uint64_t mbar;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0 && kMmaProbe) {
    // serial MMA units (4 x M=128 N=16 K=16, A from TMEM stage columns,
    // B = the first record slot as a dummy operand) + commit + wait, while
    // the decoders store into other TMEM columns
    const uint64_t bdesc = desc_kmajor_sw128(smem_u32(sm));
    const uint32_t lo = (uint32_t)bdesc, hi = (uint32_t)(bdesc >> 32);
    constexpr uint32_t IDESC = idesc_bf16_f32(128, 16);
    long long t0 = clock64();
    const int R = 512;
    for (int r = 0; r < R; ++r) {
      mma_ktile_ts(tmem, tmem + 64u + 32u * (uint32_t)(r & 7), lo, hi, IDESC, 1u, smem_u32(&mbar));
      mbar_wait(&mbar, r & 1);
    }
    long long t1 = clock64();
    if (lane == 0) cycles[gridDim.x * kDecWarps + blockIdx.x] = (t1 - t0) / R;
  }
  if (warp >= 1) {
    const int dw = warp - 1, grp = dw >> 2, q = dw & 3;
    const uint32_t lane_tm = (uint32_t)(32 * q) << 16;
    const uint32_t lut = (kVar == 2 || kVar == 3) ? smem_u32(s_lut2) : smem_u32(s_lut);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int r = (it * 4 + grp) % kR;
      const uint32_t taddr = tmem + lane_tm + 64u + 32u * (uint32_t)((it & 1) * 4 + grp);
      if (kVar == 0) decode_v0(sm + r * kSlot, taddr, q, lane, s_lut, sm);
      else if (kVar == 1) decode_v1<kVar>(smem_u32(sm + r * kSlot), taddr, q, lane, lut);
      else if (kVar == 2) decode_v2(smem_u32(sm + r * kSlot), taddr, q, lane, lut);
      else if (kVar == 4) decode_v4(smem_u32(sm + r * kSlot), taddr, q, lane, lut);
      else decode_v3(smem_u32(sm + r * kSlot), taddr, q, lane, lut);
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cycles[blockIdx.x * kDecWarps + dw] = t1 - t0;
    // correctness: group grp decodes record grp into TMEM columns 32*grp
    const uint32_t taddr = tmem + lane_tm + 320u + 32u * (uint32_t)grp;
    if (kVar == 0) decode_v0(sm + grp * kSlot, taddr, q, lane, s_lut, sm);
    else if (kVar == 1) decode_v1<kVar>(smem_u32(sm + grp * kSlot), taddr, q, lane, lut);
    else if (kVar == 2) decode_v2(smem_u32(sm + grp * kSlot), taddr, q, lane, lut);
    else if (kVar == 4) decode_v4(smem_u32(sm + grp * kSlot), taddr, q, lane, lut);
    else decode_v3(smem_u32(sm + grp * kSlot), taddr, q, lane, lut);
    tc_fence_before();
    uint32_t v[16];
    for (int h = 0; h < 2; ++h) {
      SALR_TMEM_LD_X16(taddr + 16u * h, v);
      tc_wait_ld();
      if (blockIdx.x == 0)
        for (int k = 0; k < 16; ++k) out[(grp * 128 + 32 * q + lane) * 32 + 16 * h + k] = v[k];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// host TB2 record of a random 64x128 tile; dense[col][32 words] expected TMEM words
static uint32_t make_record(std::mt19937& g, double p, uint8_t* rec, uint32_t* dense) {
  std::uniform_real_distribution<float> U(0.f, 1.f);
  uint16_t w[64][128];
  for (int k = 0; k < 64; ++k)
    for (int n = 0; n < 128; ++n) {
      if (U(g) < p) { w[k][n] = 0; continue; }
      uint16_t v;
      do { v = (uint16_t)(g() & 0xFFFF); } while ((v & 0x7F80) == 0x7F80 || v == 0 || v == 0x8000);
      w[k][n] = v;
    }
  memset(rec, 0, kSlot);
  uint32_t* hdr = reinterpret_cast<uint32_t*>(rec);
  uint16_t* bandoff = reinterpret_cast<uint16_t*>(rec + kT2BandOff);
  uint64_t* cm = reinterpret_cast<uint64_t*>(rec + kT2Mask);
  uint16_t* vals = reinterpret_cast<uint16_t*>(rec + kT2Val);
  uint32_t pos = 0;
  for (int q = 0; q < 4; ++q) {
    if (q) hdr[q - 1] = pos;
    const uint32_t gstart = pos;
    for (int b = 0; b < 16; ++b) {
      bandoff[q * 16 + b] = (uint16_t)(pos - gstart);
      for (int l = 0; l < 32; ++l)
        for (int r = 4 * b; r < 4 * b + 4; ++r)
          if (w[r][32 * q + l]) vals[pos++] = w[r][32 * q + l];
    }
    for (int l = 0; l < 32; ++l) {
      uint64_t m = 0;
      for (int r = 0; r < 64; ++r) if (w[r][32 * q + l]) m |= 1ull << r;
      cm[32 * q + l] = m;
    }
  }
  hdr[3] = pos;
  if (kT2Val + 2 * pos > kSlot) { fprintf(stderr, "record too big\n"); exit(1); }
  for (int n = 0; n < 128; ++n)
    for (int j = 0; j < 32; ++j) dense[n * 32 + j] = (uint32_t)w[2 * j][n] | ((uint32_t)w[2 * j + 1][n] << 16);
  return kT2Val + 2 * pos;
}

template <int kVar>
static void run(const uint8_t* d_recs, const uint32_t* d_rb, const std::vector<uint32_t>& dense, int iters) {
  long long* d_cyc;
  uint32_t* d_out;
  const int G = 148;
  cudaMalloc(&d_cyc, sizeof(long long) * G * (kDecWarps + 1));
  cudaMalloc(&d_out, 4 * 128 * 32 * 4);
  cudaMemset(d_out, 0, 4 * 128 * 32 * 4);
  const size_t smem = kR * kSlot;
  cudaFuncSetAttribute(bench_kernel<kVar>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench_kernel<kVar><<<G, 32 * (kDecWarps + 1), smem>>>(d_recs, d_rb, 8, d_cyc, d_out);
  bench_kernel<kVar><<<G, 32 * (kDecWarps + 1), smem>>>(d_recs, d_rb, iters, d_cyc, d_out);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("V%d: CUDA error %s\n", kVar, cudaGetErrorString(err)); exit(1); }
  std::vector<long long> cyc(G * (kDecWarps + 1));
  std::vector<uint32_t> out(4 * 128 * 32);
  cudaMemcpy(cyc.data(), d_cyc, cyc.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost);
  long long mx = 0;
  double avg = 0;
  for (int b = 0; b < G; ++b) {
    long long m = 0;
    for (int w = 0; w < kDecWarps; ++w) m = cyc[b * kDecWarps + w] > m ? cyc[b * kDecWarps + w] : m;
    mx = m > mx ? m : mx;
    avg += m;
  }
  avg /= G;
  int bad = 0;
  for (size_t i = 0; i < out.size(); ++i) bad += out[i] != dense[i];
  printf("V%d: %.1f cycles per tile per SM (avg CTA), %.1f (slowest), mismatches %d; serial MMA unit during decode: %lld cycles\n", kVar, avg / (4.0 * iters),
         (double)mx / (4.0 * iters), bad, kMmaProbe ? cyc[G * kDecWarps] : 0ll);
  cudaFree(d_cyc);
  cudaFree(d_out);
}

int main(int argc, char** argv) {
  const double p = argc > 1 ? atof(argv[1]) : 0.5;
  const int iters = 2048;
  std::mt19937 g(1234);
  std::vector<uint8_t> recs(kR * kSlot);
  std::vector<uint32_t> rb(kR);
  std::vector<uint32_t> dense_all(kR * 128 * 32);
  double bytes = 0;
  for (int r = 0; r < kR; ++r) {
    rb[r] = make_record(g, p, recs.data() + r * kSlot, dense_all.data() + r * 128 * 32);
    bytes += rb[r];
  }
  // groups 0..3 decode records 0..3 for the check
  std::vector<uint32_t> dense(4 * 128 * 32);
  memcpy(dense.data(), dense_all.data(), dense.size() * 4);
  uint8_t* d_recs;
  uint32_t* d_rb;
  cudaMalloc(&d_recs, recs.size());
  cudaMalloc(&d_rb, rb.size() * 4);
  cudaMemcpy(d_recs, recs.data(), recs.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(d_rb, rb.data(), rb.size() * 4, cudaMemcpyHostToDevice);
  printf("p=%.2f avg record %.0f B; HBM-rate budget at 6.54 TB/s, 1.965 GHz, 148 SMs: %.0f cycles per tile\n", p,
         bytes / kR, bytes / kR / (6.54e12 / 148 / 1.965e9));
  run<0>(d_recs, d_rb, dense, iters);
      run<4>(d_recs, d_rb, dense, iters);
  return 0;
}
