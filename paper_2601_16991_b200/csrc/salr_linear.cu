// SALR linear forward on sm_100a:  Y = X @ decode(W) + (X @ A_cat) @ B_cat
//
// Reference: pkg/src/salr/pipeline.py:275-331 (pipelined_forward: stage-1
// bitmap decode into tiles, stage-2 tile products, adapter delta added once),
// pkg/src/salr/fusion.py:87-92 (apply_fused: exactly two products).
//
// B200 design:
//   * swap-AB: the tensor core computes a Y^T tile = W^T tile (128 output
//     columns = M_mma 128) x X^T (N_mma = BM tokens), fp32 accumulator in TMEM.
//   * warp roles of one persistent CTA per SM (24 warps, 6 per sub-partition):
//       warps 0, 3  TMA producers (even / odd work units): each TB2 / NM24 record
//                   (1-D bulk copy, L2 evict-first) into a ring of up to 8
//                   shared-memory stages (full/empty mbarriers, expect_tx),
//                   the X tile (2-D tensor map, 128B swizzle) on its own
//                   barrier; records of the first ring go out before the
//                   programmatic-launch wait.
//       warp 1      MMA issuer (one elected lane), TMEM allocator.
//       warp 2      publisher: releases the CTA's first split-K partial;
//                   fills the decoders' nibble table at entry.
//       warps 4-19  decoders, four groups of four warps.  Group g decodes
//                   units = g (mod 4); warp (g, q) owns output columns
//                   32q..32q+31 == TMEM lanes 32q..32q+31, expands the 64
//                   rows of its column from the band runs of the TB2 record
//                   (or selects them from the NM24 record of a 2:4 matrix)
//                   and writes bf16 pairs along K with tcgen05.st straight
//                   into the TMEM A operand of the next MMA -- decoded tiles
//                   never touch shared memory.
//       warps 20-23 epilogue: in-kernel U = X @ A_cat (warp-level mma.sync,
//                   int64 fixed-point atomics), adapter operands, TMEM
//                   accumulator -> Y or an fp32 split-K partial.
//   * the ring is the GPU form of the reference's SPSC _Ring
//     (pipeline.py:110-183): decode of tile k+1 overlaps the MMA of tile k.
//   * adapters: the CTA that owns k-tile 0 of an output tile adds
//     B_cat^T x [U_hi | U_lo]^T into the SAME TMEM accumulator (two
//     SMEM-operand MMAs), so Y leaves the chip once.
//   * stream-K: every CTA owns a contiguous range of (m-chunk, n-tile, k-tile)
//     work units; split output tiles are summed in a fixed CTA order through
//     DSMEM (thread-block clusters) or global memory -- results are
//     bit-identical from run to run (the reference's schedule independence,
//     test_pipeline.py:90-112).
//   * M > 256: salr_prefill.cuh (one decode per weight tile per 512 tokens).

#include <algorithm>
#include <cstring>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "salr_format.cuh"
#include "salr_ptx.cuh"
#include "salr_status.cuh"

namespace salr {

struct LinearParams {
  const uint8_t* records;
  const uint32_t* tile_off;
  void* y;
  float* partials;    // [2 * gridDim.x][BM][128] fp32 split-K partial tiles
  uint32_t* tickets;  // n_mc * n_nt, zero on entry and exit
  int M, N, ldy;      // 32-bit indexing: host checks M * max(N, ldy) < 2^31
  int n_kt, n_nt, n_mc;
  int units;          // n_mc * n_nt * n_kt
  int ra;             // adapter rank blocks of 64 (0 = no adapters)
  int u_mode;         // 1 = U computed in-kernel (fixed-point atomics), 2 = U hi/lo from the pre-kernel
  int K;              // d_in (for the in-kernel U slices)
  const __nv_bfloat16* x;      // X (M x K, ld ldx) for the in-kernel U
  const __nv_bfloat16* acat;   // A_cat (K x 64*ra) for the in-kernel U
  int ldx;
  unsigned long long* u_acc;   // [2][M][64*ra] int64 fixed point (2^kUFrac), parity-buffered
  uint32_t* ctrl;              // adapter control words (fixed workspace offset)
  int y_dtype;
  int stages;         // ring slots in use
  int coop;           // 1: grid <= SM count, split tiles are reduced cooperatively
  int cluster;        // > 1: every output tile is split over exactly the `cluster`
                      // CTAs of one thread-block cluster; reduced through DSMEM
  uint32_t rec_slot;  // bytes per ring slot: the largest record of this matrix, 16-aligned
  int nm24;           // 1: records are NM24 (fixed kNmRecBytes per tile, tile_off unused)
  int dbg;            // timing experiments only: 1 = skip decode, 2 = skip record loads
  unsigned long long* trace;  // optional per-CTA event timestamps (globaltimer ns), [G][32]
  // Pipeline probe (salr_debug_set_probe; null = off): device form of the
  // reference PipelineProbe (pipeline.py:89-103).  log[0] = entries,
  // log[1] = produced, log[2] = consumed, log[4 + i] = slot << 8 | old << 4 |
  // new for the slot (cta * S + stage) transitions EMPTY(0) -> FILLED(1) ->
  // CONSUMED(2) -> EMPTY, and each decode / MMA issue sleeps a hashed
  // 0..probe_ns ns first (fault injection by jitter).
  uint32_t* probe_log;
  uint32_t probe_cap;
  uint32_t probe_ns;
  uint32_t probe_seed;
  // shared-memory carve-up (bytes from the 1024-aligned base)
  uint32_t x_off, rec_off, base_off, ad_off, bar_off;
};

// In-kernel U = X @ A_cat: CTAs claim K slices and add their partials into an
// int64 fixed-point accumulator (2^-kUFrac resolution).  Integer addition is
// associative, so U is bit-reproducible whatever the CTA order.
constexpr int kUFrac = 26;
// ctrl words: [0] epoch (parity selects the U buffer), [1] done counter,
// [2..3] slices done[parity], [4..5] used elements of u_acc[parity],
// [6..7] slice claim counter[parity]
constexpr int kCtrlEpoch = 0, kCtrlDone = 1, kCtrlReady = 2, kCtrlUsed = 4, kCtrlSlice = 6;
constexpr int kUSlice = 64;  // K rows per dynamically claimed U slice
constexpr int kDoneTicketOff = 16 * 1024;  // second counter per split tile (workspace ticket area)
constexpr int kUAccElems = 256 * 128;  // per parity buffer: M <= 256 rows x r_pad <= 128
constexpr int kNumDecWarps = 16;
// The odd-unit producer runs on warp 3 (sub-partition 3, otherwise idle):
// with it on a 25th warp, sub-partition 0 hosted both producers next to four
// decoder warps and an epilogue warp, and its decoders lagged the group by
// ~1 us per tile (unit traces).  The block size only sets the register
// budget then: 24 warps (80 registers) for BM = 16 tiles, 25 (72 registers,
// warp 24 idle) for larger ones -- measured best per tile size on the
// 32-layer stack (A/B, tools/gpu_ab_bench.sh).
#ifndef SALR_PROD1_WARP
#define SALR_PROD1_WARP 3
#endif
__host__ __device__ constexpr int threads_for(int bm) {
#ifdef SALR_NUM_WARPS
  return 32 * SALR_NUM_WARPS + 0 * bm;
#else
  return (SALR_PROD1_WARP == 3 && bm == 16) ? 768 : 800;
#endif
}
constexpr int kFirstDecWarp = 4;
constexpr int kFirstEpiWarp = 20;
// warp layout helpers of the chained-linear kernel (salr_chain.cuh): NG
// decoder groups of four warps after warps 0-3, then four epilogue warps
__host__ __device__ constexpr int first_epi_warp(int ng) { return kFirstDecWarp + 4 * ng; }
__host__ __device__ constexpr int num_threads(int ng) { return 32 * (first_epi_warp(ng) + 4); }
constexpr uint32_t kAdTileBytes = 128 * 128;   // B_cat^T tile: 128 rows x 64 bf16
constexpr size_t kSmemMax = 232448;            // 227 KB opt-in per block
constexpr size_t kSmemMaxLinear = kSmemMax - 128;  // minus the decoders' static nibble table
constexpr int64_t kPrefillMinM = 256;          // M above this: salr_prefill_kernel

__host__ __device__ constexpr int nacc_for(int bm) { return bm <= 128 ? 2 : 1; }
__host__ __device__ constexpr int acc_cols_for(int bm) { return bm < 32 ? 32 : bm; }

struct SmemPlan {
  uint32_t x_off, rec_off, base_off, ad_off, bar_off, total;
};

// Nibble expansion table of the decoder.  For the 4-bit column mask n of a
// 4-row band (bit i = row i present) whose values start at byte address r:
//   word 0 (rows 0,1) = prmt(v[r],    v[r+2],    sel(n & 3))
//   word 1 (rows 2,3) = prmt(v[r+2c], v[r+2c+2], sel(n >> 2)),  c = popc(n & 3)
// with each v[] loaded zero-extended to 32 bits, so bytes 2,3 of the first
// source are zero: sel(00) = 0x3232 (0), sel(01) = 0x3210 ([v, 0]),
// sel(10) = 0x1032 ([0, v]), sel(11) = 0x5410 ([v, v']).  Entry =
// sel(n & 3) | (2c) << 16 (low word; prmt reads only bits 0-15) and
// sel(n >> 2) (high word).
__host__ __device__ constexpr uint32_t nib_sel(uint32_t x) {
  return x == 0 ? 0x3232u : x == 1 ? 0x3210u : x == 2 ? 0x1032u : 0x5410u;
}
__host__ __device__ constexpr uint64_t nib_lut_entry(uint32_t n) {
  return (uint64_t)(nib_sel(n & 3u) | ((2u * ((n & 1u) + ((n >> 1) & 1u))) << 16)) |
         ((uint64_t)nib_sel(n >> 2) << 32);
}
// stage-dependent layout; 1024-aligned pieces first (swizzled TMA/UMMA tiles)
__host__ __device__ inline SmemPlan smem_plan(int bm, int stages, int ra, uint32_t rec_slot) {
  SmemPlan p;
  p.ad_off = 0;                                            // ra x (Bcat tile + U hi + U lo)
  const uint32_t ad_bytes = (uint32_t)ra * (kAdTileBytes + 2u * bm * 128u);
  p.x_off = p.ad_off + ad_bytes;                           // stages x BM x 128 B
  p.rec_off = p.x_off + (uint32_t)stages * bm * 128u;      // stages x kRecSlot
  p.base_off = p.rec_off + (uint32_t)stages * rec_slot;    // stages x 256 u32
  p.bar_off = p.base_off;
  p.total = p.bar_off + 8u * (4u * stages + 6u) + 16u + 1024u;  // + tmem slot + alignment slack
  return p;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// ---- pipeline probe helpers (see LinearParams::probe_log)
enum : uint32_t { kSlotEmpty = 0, kSlotFilled = 1, kSlotConsumed = 2 };
__device__ __forceinline__ void probe_log_transition(uint32_t* log, uint32_t cap, uint32_t slot, uint32_t from,
                                                     uint32_t to) {
  const uint32_t i = atomicAdd(log, 1u);
  if (i < cap) log[4 + i] = slot << 8 | from << 4 | to;
  if (from == kSlotEmpty) atomicAdd(log + 1, 1u);
  if (from == kSlotFilled) atomicAdd(log + 2, 1u);
  __threadfence();
}
__device__ __forceinline__ void probe_jitter(uint32_t ns, uint32_t seed, uint32_t a, uint32_t b) {
  if (!ns) return;
  uint32_t h = seed ^ (a * 0x9E3779B9u) ^ (b * 0x85EBCA6Bu);
  h ^= h >> 16;
  h *= 0x7FEB352Du;
  h ^= h >> 15;
  __nanosleep(h % (ns + 1));
}

// per-unit detail for CTA 0 (first 64 units): slot 148*32 + ev*64 + i
// (compiled in only with -DSALR_UNIT_TRACE: the stamps sit in the per-unit
// hot loops, where even predicated-off instructions cost issue slots)
#ifdef SALR_UNIT_TRACE
#define SALR_TRACE_UNIT(ev, i)                                                               \
  do {                                                                                       \
    if (p.trace && blockIdx.x == 0 && (i) < 64) p.trace[148 * 32 + (ev) * 64 + (i)] = clock64(); \
  } while (0)
#else
#define SALR_TRACE_UNIT(ev, i) \
  do {                         \
  } while (0)
#endif
#define SALR_TRACE(ev) \
  do {                 \
    if (p.trace) p.trace[(size_t)blockIdx.x * 32 + (ev)] = globaltimer(); \
  } while (0)

// CTA that owns work unit u under the even contiguous split of `units` over `ctas`.
__device__ __forceinline__ int cta_of(int u, int units, int ctas) {
  return (int)((((int64_t)u + 1) * ctas + units - 1) / units - 1);
}

// acq_rel ticket: orders this thread's prior (fenced-by-CTA-barrier) writes
// before the increment and the reads after it behind it, at GPU scope.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* addr) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t saddr, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(saddr), "r"(rank));
  float4 v;
  // volatile: stays behind the cluster barrier (also a volatile asm); the
  // caller issues every rank's load before the first use
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra));
  return v;
}
// acquire-release fence at GPU scope (release/acquire patterns with relaxed
// atomics).  (__threadfence() is the sequentially consistent fence.)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ticket_add_acq_rel(uint32_t* addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(addr), "r"(v) : "memory");
  return old;
}

// Warp roles (see the file header).  Every mbarrier hand-off costs ~150-300
// SM cycles of latency on B200 (measured, tools/ubench/ubench_sync.cu), so
// each serial role is split across warps that work on different units
// concurrently: two producers (even / odd units), two row-base warps, and
// TB2 tile decoder, one warp: TMEM lane quarter q (output columns 32q..32q+31),
// all 64 rows.  Per lane (one output column) and 4-row band the values are
// contiguous: the band's run starts at bandoff[q][b] + (exclusive warp prefix
// of the band counts), and four zero-extended loads plus two byte permutes
// driven by the nibble table expand the 4 rows -- no per-element rank
// popcounts.  Writes the lane's 32 bf16-pair columns of the A operand with
// tcgen05.st (the caller waits and fences).
// (BPW < 16: bands [BPW * part, BPW * part + BPW) only, a decoder group of
// more than four warps splitting the rows; taddr then points at that part.)
template <int BPW = 16>
__device__ __forceinline__ void decode_tile_tb2(uint32_t rec_s, uint32_t taddr, int q, uint32_t lane,
                                                uint32_t lut_s, int part = 0) {
  const uint2 mw = lds_v2_u32(rec_s + kT2Mask + 8u * (32u * q + lane));
  // 4-bit band counts as bytes: c[0] bands 0,2,4,6; c[1] 1,3,5,7;
  // c[2] 8,10,12,14; c[3] 9,11,13,15
  uint32_t nl = mw.x - ((mw.x >> 1) & 0x55555555u);
  uint32_t nh = mw.y - ((mw.y >> 1) & 0x55555555u);
  nl = (nl & 0x33333333u) + ((nl >> 2) & 0x33333333u);
  nh = (nh & 0x33333333u) + ((nh >> 2) & 0x33333333u);
  const uint32_t c[4] = {nl & 0x0F0F0F0Fu, (nl >> 4) & 0x0F0F0F0Fu, nh & 0x0F0F0F0Fu, (nh >> 4) & 0x0F0F0F0Fu};
  uint32_t e[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {  // inclusive scan, byte lanes (<= 128)
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
  const uint32_t goff = q ? lds_u32(rec_s + 4u * (uint32_t)(q - 1)) : 0u;
  const uint32_t vb = rec_s + kT2Val + 2u * goff;
  const uint4 bo0 = lds_v4_u32(rec_s + kT2BandOff + 32u * q);
  const uint4 bo1 = lds_v4_u32(rec_s + kT2BandOff + 32u * q + 16u);
  const uint32_t bo[8] = {bo0.x, bo0.y, bo0.z, bo0.w, bo1.x, bo1.y, bo1.z, bo1.w};
#pragma unroll
  for (int pp = 0; pp < 16 / BPW; ++pp) {  // this warp's part, unrolled so bands are compile-time
    if (pp != part) continue;
#pragma unroll
  for (int c4 = 0; c4 < BPW / 4; ++c4) {  // 4 bands -> 8 TMEM columns
    uint32_t packed[8];
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const int b = BPW * pp + 4 * c4 + i;  // bands b, b+1
      // byte offsets of both bands' runs in 16-bit lanes: (prefix + band
      // offset) * 2; byte prefixes are < 128, so sign-replicating selector
      // nibbles give the zero bytes
      const int j = (b & 7) >> 1;
      const uint32_t pe = prmt(e[b >= 8 ? 2 : 0], e[b >= 8 ? 3 : 1],
                               (uint32_t)j | ((0x8u | j) << 4) | ((4u + j) << 8) | ((0x8u | j) << 12));
      const uint32_t pr2 = pe + pe + (bo[b >> 1] + bo[b >> 1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bb = b + h;
        const uint32_t r = h ? vb + (pr2 >> 16) : vb + (pr2 & 0xFFFFu);
        const int sh = 4 * (bb & 7);
        const uint32_t word = bb < 8 ? mw.x : mw.y;
        // nibble -> table entry (8 bytes): selectors of both row pairs and
        // the byte offset of pair 1's first value.  Absent elements need no
        // predicate: the selectors pick zero bytes of the zero-extended loads.
        const uint32_t nib8 = (sh >= 3 ? (word >> (sh - 3)) : (word << 3)) & 0x78u;
        const uint2 ent = lds_v2_u32(lut_s | nib8);
        const uint32_t r2 = r + (ent.x >> 16);
        const uint32_t a0 = lds_u16z(r), a1 = lds_u16z(r + 2u);
        const uint32_t b0 = lds_u16z(r2), b1 = lds_u16z(r2 + 2u);
        packed[2 * (i + h)] = prmt(a0, a1, ent.x);
        packed[2 * (i + h) + 1] = prmt(b0, b1, ent.y);
      }
    }
    SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
  }
  }
}

// NM24 tile decoder (salr_format.cuh), same TMEM result as decode_tile_tb2.
// Lane = output column 32q + lane = column j of 4-column group g.  Per 8 rows
// one mask word gives, as bit 7 of byte p, "row 2p (<<4) / 2p+1 kept in
// column j" and "a lower column of the group is kept too" (then this column
// holds the group's second value v1): sign-replicating permutes turn those
// bits into the byte mask and the value selector of the row pair.
template <int BPW = 16>
__device__ __forceinline__ void decode_tile_nm24(uint32_t rec_s, uint32_t taddr, int q, uint32_t lane, int part = 0) {
  const uint32_t g = 8u * (uint32_t)q + (lane >> 2), j = lane & 3u;
  const uint32_t lower = 0x11111111u * ((1u << j) - 1u);  // columns below j, every nibble
  const uint32_t sh = 3u - j;
#pragma unroll
  for (int pp = 0; pp < 16 / BPW; ++pp) {
    if (pp != part) continue;
#pragma unroll
    for (int c4 = 0; c4 < BPW / 4; ++c4) {
      const int b0 = BPW * pp + 4 * c4;  // bands b0..b0+3 = rows 4*b0 .. 4*b0+15
      const uint2 mw = lds_v2_u32(rec_s + kNmValBytes + 16u * (32u * (uint32_t)(b0 >> 3) + g) +
                                  4u * (uint32_t)((b0 >> 1) & 3));
      uint32_t packed[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // mask word h: bands b0 + 2h, b0 + 2h + 1
        const uint32_t m = h ? mw.y : mw.x;
        const uint32_t kx = (m << sh) & 0x88888888u;                     // kept, bit 4i+3
        const uint32_t bx = ((m & lower) + 0x77777777u) & 0x88888888u;  // second value
        const uint32_t klo = kx << 4, blo = bx << 4;
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          const uint4 w = lds_v4_u32(rec_s + 16u * (32u * (uint32_t)(b0 + 2 * h + bb) + g));
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t pidx = 2u * bb + t;  // row pair within the mask word
            // byte mask of the pair (16-bit halves) and the value selector
            // (nibble pairs: +2 picks v1's bytes)
            const uint32_t sel = (0x8u | pidx) * 0x11u | ((0xCu | pidx) * 0x11u) << 8;
            const uint32_t vsel = (0x8u | pidx) | (0xCu | pidx) << 4;
            const uint32_t msk = prmt(klo, kx, sel);
            const uint32_t vs = (prmt(blo, bx, vsel) & 0x2222u) | 0x5410u;
            packed[4 * h + 2 * bb + t] = prmt(t ? w.z : w.x, t ? w.w : w.y, vs) & msk;
          }
        }
      }
      SALR_TMEM_ST_X8(taddr + 8u * c4, packed);
    }
  }
}

// kDecGroups decoder groups (group g decodes units it = g mod kDecGroups).
constexpr int kWarpProd0 = 0, kWarpMma = 1, kWarpPub = 2;
constexpr int kWarpProd1 = SALR_PROD1_WARP;

template <int BM, int kDecGroups, bool kProbe = false>
__global__ void __launch_bounds__(threads_for(BM), 1)
    salr_linear_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap bmap,
                       const __grid_constant__ CUtensorMap uhimap, const __grid_constant__ CUtensorMap ulomap,
                       const LinearParams p) {
  constexpr int NACC = nacc_for(BM);
  constexpr int ACOLS = acc_cols_for(BM);
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BM);
  constexpr int WPG = kNumDecWarps / kDecGroups;  // decoder warps per group
  constexpr int RPW = 4 * kTileK / WPG;           // rows per decoder warp (all 4 lane quarters per group)

  extern __shared__ uint8_t smem_raw[];
  // 128B-swizzled TMA/UMMA tiles need 1024-byte alignment; pad by an offset
  // (not a pointer round-trip) so the compiler keeps the shared address space.
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const int S = p.stages;
  uint8_t* xbuf = smem + p.x_off;
  uint8_t* recbuf = smem + p.rec_off;
  uint8_t* adbuf = smem + p.ad_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + S;
  uint64_t* decoded = empty + S;
  // X tiles complete on their own barriers: the decoders wait only for the
  // records, which are in flight before the programmatic-launch wait, so
  // they decode the first ring while the preceding kernel drains; the MMA
  // waits for both
  uint64_t* xfull = decoded + S;
  uint64_t* acc_full = xfull + S;      // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint64_t* ad_full = acc_empty + 2;
  uint64_t* ad_empty = ad_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ad_empty + 1);
  volatile uint32_t* last_flag = tmem_slot + 1;
  uint32_t* zero_word = tmem_slot + 2;  // a shared zero the decoders load for absent elements
  volatile uint32_t* early_old_slot = tmem_slot + 3;  // publisher warp -> epilogue

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) SALR_TRACE(10);
  // let the next kernel in the stream start its weight-only prologue as soon
  // as SMs free up (it waits for this grid before touching our output)
  if (threadIdx.x == 0) pdl_launch_dependents();
  if (threadIdx.x == 0 && p.trace && blockIdx.x == 0) p.trace[148 * 32 + 7 * 64] = clock64();

  // ---- per-CTA work range
  const int G = gridDim.x;
  const int u_begin = (int)((int64_t)blockIdx.x * p.units / G);
  const int u_end = (int)(((int64_t)blockIdx.x + 1) * p.units / G);
  const int tiles_per_mc = p.n_nt * p.n_kt;
  // The CTA's first segment is a split tile with more work behind it: its
  // partial is published mid-run by the publisher warp (see the epilogue).
  const int first_seg_end0 = min(u_end, u_begin - u_begin % p.n_kt + p.n_kt);
  const bool early_split = !p.cluster && (u_begin % p.n_kt != 0 || first_seg_end0 - u_begin < p.n_kt) &&
                           first_seg_end0 < u_end;

  // ---- producer state (warps kWarpProd0 / kWarpProd1, units of one parity).
  // Record offsets are fetched 32 units at a time, one chunk ahead, one
  // coalesced load per lane, so the issue loop never waits on a global load.
  // Each multi-instance role owns the stages s = instance (mod instances), so
  // an instance never waits on a stage two phases ahead (mbarrier parity
  // waits cannot tell those apart): the host picks S as a multiple of the
  // decoder group count, and the producers / row-base warps run as pairs only
  // when S is even.
  const int NP = (S % 2 == 0) ? 2 : 1;
  const int pk = warp == kWarpProd1 ? 1 : 0;
  uint32_t co0 = 0, co1 = 0, no0 = 0, no1 = 0;
  int chunk = u_begin;
  int pv = u_begin + pk;  // next unit to issue (this producer's parity)
  int ps = pk;            // < S whenever this producer is active
  uint32_t pph = 0;
  const uint64_t pol_stream = l2_policy_evict_first();
  auto load_chunk = [&](int c0, uint32_t& o0, uint32_t& o1) {
    const int v = c0 + (int)lane;
    o0 = o1 = 0u;
    if (v < u_end) {
      const int t = v % tiles_per_mc;
      if (p.nm24) {
        o0 = (uint32_t)t * (kNmRecBytes / 16);
        o1 = o0 + kNmRecBytes / 16;
      } else {
        o0 = __ldg(p.tile_off + t);
        o1 = __ldg(p.tile_off + t + 1);
      }
    }
  };
  // X tile of unit v into stage st (the input; may have to wait for the
  // preceding kernel under programmatic dependent launch)
  // The X tile lands on the stage's `decoded` barrier (one producer arrival
  // + its bytes next to the decoder warps' arrivals), so the MMA issuer --
  // the CTA's serial path -- waits on one barrier per unit.
  auto issue_x = [&](int v, int st) {
    if (p.dbg & 16) {  // experiment: no X tiles
      mbar_arrive(&decoded[st]);
      return;
    }
    const int kt = v % p.n_kt;
    const int mc = v / tiles_per_mc;
    tma_2d_g2s(xbuf + (size_t)st * BM * 128, &xmap, kt * kTileK, mc * BM, &decoded[st]);
    mbar_arrive_expect_tx(&decoded[st], BM * 128);
  };
  // Issue unit pv.  The copies go out before arrive.expect_tx (the phase
  // cannot complete before the arrive, and issuing the copy first keeps it
  // off the arrive's latency).  The first ring's worth of units never waits
  // for `empty`.  with_x = false defers the X tile (see the PDL prologue).
  auto issue_one = [&](bool with_x) {
    if (lane == 0) SALR_TRACE_UNIT(8, pv - u_begin);
    while (pv - chunk >= 32) {
      chunk += 32;
      co0 = no0;
      co1 = no1;
      load_chunk(chunk + 32, no0, no1);
    }
    const uint32_t o0 = __shfl_sync(0xffffffffu, co0, pv - chunk);
    const uint32_t o1 = __shfl_sync(0xffffffffu, co1, pv - chunk);
    if (lane == 0) SALR_TRACE_UNIT(9, pv - u_begin);
    if (pv - u_begin >= S) {
      mbar_wait(&empty[ps], pph ^ 1);
      if (kProbe && lane == 0)
        probe_log_transition(p.probe_log, p.probe_cap, (uint32_t)(blockIdx.x * S + ps), kSlotConsumed, kSlotEmpty);
    }
    if (lane == 0) {
      SALR_TRACE_UNIT(10, pv - u_begin);
      const uint32_t bytes = (p.dbg & 2) ? 0u : (o1 - o0) * 16u;
      if (bytes) bulk_g2s_hint(recbuf + (size_t)ps * p.rec_slot, p.records + (size_t)o0 * 16u, bytes, &full[ps], pol_stream);
      mbar_arrive_expect_tx(&full[ps], bytes);
      if (with_x) issue_x(pv, ps);
      SALR_TRACE_UNIT(0, pv - u_begin);
    }
    __syncwarp();
    ps += NP;
    if (ps >= S) { ps -= S; pph ^= 1; }
    pv += NP;
  };

  const bool producer = warp == kWarpProd0 || (warp == kWarpProd1 && NP == 2);
  if (warp == kWarpProd0 || warp == kWarpProd1) {
    load_chunk(u_begin, co0, co1);
    load_chunk(u_begin + 32, no0, no1);
    if (warp == kWarpProd0 && lane == 0) {
      prefetch_tmap(&xmap);
      if (p.ra) {
        prefetch_tmap(&bmap);
        prefetch_tmap(&uhimap);
        prefetch_tmap(&ulomap);
      }
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&xfull[s], 1);
        mbar_init(&empty[s], 1);
        mbar_init(&decoded[s], WPG + 1);  // decoder warps + the X tile's producer
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&acc_full[b], 1);
        mbar_init(&acc_empty[b], 4);
      }
      mbar_init(ad_full, 1);
      mbar_init(ad_empty, 1);
      *zero_word = 0u;
      fence_barrier_init();
    }
    named_bar_sync(2, 64);  // barriers initialised before either producer uses them
    if (threadIdx.x == 0) SALR_TRACE(21);
    // Start streaming before the CTA-wide setup barrier: this producer's share
    // of the first ring's worth of units of the first output tile (never blocks).
    const int first_seg_end = min(u_end, u_begin - u_begin % p.n_kt + p.n_kt);
    const int pre = min(first_seg_end, u_begin + S);
    if (producer)
      while (pv < pre) issue_one(false);
    if (threadIdx.x == 0) SALR_TRACE(23);
  }
  // ---- in-kernel U (u_mode 1) geometry.  K is cut into slices of kUSlice
  // rows.  CTA c owns slice c; slices >= G are claimed dynamically.  A_cat is
  // a weight, so the A rows of the owned slice are copied into the (still
  // unused) adapter slot before waiting for the preceding kernel, and the
  // dynamically claimed ones are prefetched into L2.  (Everything U-related
  // is recomputed where used: nothing stays live across the decode loops.)
  constexpr int kSX = kUSlice + 8;  // X chunk row stride (pads: conflict-free
  auto u_geom_wide = [&]() { return (p.dbg & 4) ? false : ((u_end - u_begin) < 8 && p.M >= 16); };
  auto u_kSA = [&]() { return 64 * p.ra + 8; };  // A slice row stride   mma fragment loads)
  auto u_staged_fn = [&]() {
    return (p.K % 8 == 0) &&
           (uint32_t)(kUSlice * u_kSA() + BM * kSX) * 2u <= (uint32_t)p.ra * (kAdTileBytes + 2u * BM * 128u);
  };
  // stage A rows of slice sl (zero rows past K, up to a whole mma k-step)
  auto u_load_a = [&](int sl, int ut, int nthr) {
    const int rp = 64 * p.ra, kSA = u_kSA();
    __nv_bfloat16* const sa = reinterpret_cast<__nv_bfloat16*>(adbuf);
    const int k0 = sl * kUSlice, ks = min(kUSlice, p.K - k0), ks16 = (ks + 15) & ~15;
    const int cpr = rp / 8;  // 16-byte chunks per row
    const __nv_bfloat16* src = p.acat + (size_t)k0 * rp;
    for (int i = ut; i < ks16 * cpr; i += nthr) {
      const int kr = i / cpr, c = i % cpr;
      cp_async_16(smem_u32(sa + kr * kSA + 8 * c), src + (size_t)(kr < ks ? i : 0) * 8, kr < ks ? 16u : 0u);
    }
  };
  if (p.u_mode == 1) {
    const bool wide = u_geom_wide();
    if (warp >= (wide ? kFirstDecWarp : kFirstEpiWarp) && warp < kFirstEpiWarp + 4 && u_staged_fn()) {
      const int ut = (warp - (wide ? kFirstDecWarp : kFirstEpiWarp)) * 32 + (int)lane;
      const int nsl = (p.K + kUSlice - 1) / kUSlice;
      if ((int)blockIdx.x < nsl) u_load_a((int)blockIdx.x, ut, wide ? 640 : 128);
      const int pf = G + (int)blockIdx.x;  // a slice another CTA may claim
      if (ut == 0 && pf < nsl)
        prefetch_l2_bulk(p.acat + (size_t)pf * kUSlice * 64 * p.ra,
                         (uint32_t)(min(kUSlice, p.K - pf * kUSlice) * 64 * p.ra * 2));
    }
  }
  // nibble table of the decoders: static shared memory, so its address is a
  // compile-time constant folded into the decoders' loads
  __shared__ __align__(128) uint64_t s_lut[16];
  if (warp == (kWarpProd1 == 3 ? kWarpPub : 3) && lane < 16) s_lut[lane] = nib_lut_entry(lane);
  const uint32_t lut_s = smem_u32(s_lut);
  if (warp == kWarpMma) {
    tmem_alloc(tmem_slot, 512);
    if (lane == 0) SALR_TRACE(27);
  }
  if (threadIdx.x == 32 * kFirstDecWarp) SALR_TRACE(16);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0u) __trap();  // all 512 columns are ours: the MMA issuer assumes base 0
  if (threadIdx.x == 0) SALR_TRACE(0);
  constexpr uint32_t a_col0 = (uint32_t)((NACC * ACOLS + 31) & ~31);  // first A-stage column

  // ---- in-kernel U = X @ A_cat (u_mode 1): each slice partial goes into
  // the int64 fixed-point accumulator (integer atomics: order-independent,
  // bit-reproducible) and is published at once (slices-done counter).
  // Participants: the epilogue warps, plus the decoder warps when a CTA has
  // fewer than 8 units and M >= 16 (work-bound partials, little decode to
  // delay; measured: with 16 units per CTA the decoders are better off
  // starting to decode).
  const bool u_wide = u_geom_wide();
  const int kUThreads = u_wide ? 640 : 128;
  if (p.u_mode == 1 && warp >= (u_wide ? kFirstDecWarp : kFirstEpiWarp) && warp < kFirstEpiWarp + 4) {
    const int ut = (warp - (u_wide ? kFirstDecWarp : kFirstEpiWarp)) * 32 + (int)lane;
    const int rp = 64 * p.ra;
    const int kSA = u_kSA();
    pdl_wait();  // X may be the preceding kernel's output
    const uint32_t par = *reinterpret_cast<volatile uint32_t*>(p.ctrl + kCtrlEpoch) & 1u;
    unsigned long long* uacc = p.u_acc + (size_t)par * kUAccElems;
    if (ut == 0) SALR_TRACE(19);
    if (blockIdx.x == 0) {
      // the previous adapter launch's buffer (other parity) is idle in this
      // launch: clear exactly the prefix its user recorded, reset its counters
      unsigned long long* other = p.u_acc + (size_t)(par ^ 1u) * kUAccElems;
      const uint32_t used = p.ctrl[kCtrlUsed + (par ^ 1u)];
      for (uint32_t i = (uint32_t)ut; i < used; i += kUThreads) other[i] = 0ull;
      if (ut == 0) {
        p.ctrl[kCtrlReady + (par ^ 1u)] = 0u;
        p.ctrl[kCtrlSlice + (par ^ 1u)] = 0u;
        p.ctrl[kCtrlUsed + (par ^ 1u)] = 0u;
        p.ctrl[kCtrlUsed + par] = (uint32_t)(p.M * rp);
      }
    }
    const int nsl = (p.K + kUSlice - 1) / kUSlice;
    const bool staged = u_staged_fn();
    __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(adbuf);
    __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(adbuf + (uint32_t)kUSlice * kSA * 2u);
    const int kURowGroups = kUThreads / 64;
    const int rg = ut >> 6;  // row group 0..kURowGroups-1 (scalar path)
    uint32_t done = 0;
    int sl = (int)blockIdx.x;  // owned slice (A rows already in flight)
    for (;;) {
      if (ut == 0 && done == 0) SALR_TRACE(15);
      if (sl >= nsl) break;
      const int k0 = sl * kUSlice, ks = min(kUSlice, p.K - k0);
      if (staged) {
        const int ks16 = (ks + 15) & ~15;  // zero-padded to whole mma k-steps
        if (done > 0) u_load_a(sl, ut, kUThreads);
        const int wid = ut >> 5, nw = kUThreads / 32;
        const int g = (int)lane >> 2, t = (int)lane & 3;
        const uint32_t sa_u = smem_u32(sa), sx_u = smem_u32(sx);
        for (int m0 = 0; m0 < p.M; m0 += BM) {
          const int rows = min(BM, p.M - m0);
          if (m0) named_bar_sync(3, kUThreads);  // previous chunk consumed
          for (int i = ut; i < rows * (ks16 / 8); i += kUThreads) {
            const int m = i / (ks16 / 8), c = i % (ks16 / 8);
            cp_async_16(smem_u32(sx + m * kSX + 8 * c),
                        p.x + (size_t)(m0 + m) * p.ldx + k0 + (c < ks / 8 ? 8 * c : 0), c < ks / 8 ? 16u : 0u);
          }
          cp_async_wait_all();
          named_bar_sync(3, kUThreads);
          if (ut == 0 && done == 0 && m0 == 0) SALR_TRACE(16);
          // (16-row block, 8-column block) items over the warps; rows past
          // `rows` read stale shared memory and are never stored.
          const int nnb = rp / 8, items = nnb * ((rows + 15) / 16);
          for (int it = wid; it < items; it += nw) {
            const int nb = it % nnb, mb = it / nnb;
            float c[4] = {0.f, 0.f, 0.f, 0.f};
            // fragments by ldmatrix: X rows (lane & 15) at k + 8 (lane >> 4);
            // A_cat k rows (lane & 15), transposed into the col-major B operand
            const uint32_t xa = sx_u + (uint32_t)(((mb * 16 + (int)(lane & 15)) * kSX + 8 * (int)(lane >> 4)) * 2);
            const uint32_t aa = sa_u + (uint32_t)(((int)(lane & 15) * kSA + nb * 8) * 2);
            for (int kk = 0; kk < ks16; kk += 16) {
              uint32_t af[4], bf[2];
              asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                           : "=r"(af[0]), "=r"(af[1]), "=r"(af[2]), "=r"(af[3])
                           : "r"(xa + (uint32_t)kk * 2));
              asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                           : "=r"(bf[0]), "=r"(bf[1])
                           : "r"(aa + (uint32_t)kk * kSA * 2));
              mma_m16n8k16_bf16(c, af, bf);
            }
            const int r0 = mb * 16 + g, n = nb * 8 + 2 * t;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int r = r0 + 8 * h;
              if (r < rows) {
                unsigned long long* dst = uacc + (size_t)(m0 + r) * rp + n;
                atomicAdd(dst, (unsigned long long)__float2ll_rn(c[2 * h] * (float)(1ll << kUFrac)));
                atomicAdd(dst + 1, (unsigned long long)__float2ll_rn(c[2 * h + 1] * (float)(1ll << kUFrac)));
              }
            }
          }
        }
      } else {
        for (int a = 0; a < p.ra; ++a) {
          const int r = 64 * a + (ut & 63);
          for (int mb = rg; mb < p.M; mb += 8 * kURowGroups) {
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
            for (int k = k0; k < k0 + ks; ++k) {
              const float av = __bfloat162float(p.acat[(size_t)k * rp + r]);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int m = mb + kURowGroups * i;
                if (m < p.M) acc[i] = fmaf(__bfloat162float(p.x[(size_t)m * p.ldx + k]), av, acc[i]);
              }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int m = mb + kURowGroups * i;
              if (m < p.M)
                atomicAdd(uacc + (size_t)m * rp + r,
                          (unsigned long long)__double2ll_rn((double)acc[i] * (double)(1ll << kUFrac)));
            }
          }
        }
      }
      ++done;
      if (ut == 0 && done == 1) SALR_TRACE(17);
      named_bar_sync(3, kUThreads);  // every partial of this slice issued; staging reusable
      if (ut == 0) {
        fence_acq_rel_gpu();
        atomicAdd(p.ctrl + kCtrlReady + par, 1u);  // consumers wait for all slices
        if (done == 1) SALR_TRACE(18);
        // next slice: dynamic claims hand out slices G, G+1, ...
        *last_flag = (uint32_t)G + atomicAdd(p.ctrl + kCtrlSlice + par, 1u);
      }
      named_bar_sync(3, kUThreads);
      sl = (int)*last_flag;
      named_bar_sync(3, kUThreads);
    }
    if (ut == 0 && done) SALR_TRACE(13);
  }

  if (warp == kWarpProd0 || warp == kWarpProd1) {
    // ================= TMA producers.  Weights never depend on the preceding
    // kernel; the input X may (it can be that kernel's output): wait for it
    // only now -- after the CTA-wide setup, so the decoders already work on
    // the first ring -- then send the X tiles of the units already in flight.
    pdl_wait();
    if (threadIdx.x == 0) SALR_TRACE(24);
    if (lane == 0 && producer) {
      const int first_seg_end = min(u_end, u_begin - u_begin % p.n_kt + p.n_kt);
      const int pre = min(first_seg_end, u_begin + S);
      for (int v = u_begin + pk; v < pre; v += NP) issue_x(v, (v - u_begin) % S);
    }
    __syncwarp();
    if (threadIdx.x == 0) SALR_TRACE(28);
    if (lane == 0 && pk == 0) SALR_TRACE(1);
    if (producer)
      while (pv < u_end) issue_one(true);
    if (kProbe && producer) {
      // probe shutdown: every slot of this producer returns to EMPTY (its
      // last MMA completes)
      for (int v = max(u_begin, u_end - S); v < u_end; ++v) {
        if ((v - u_begin) % NP != pk) continue;
        const int st = (v - u_begin) % S;
        mbar_wait(&empty[st], (uint32_t)(((v - u_begin) / S) & 1));
        if (lane == 0)
          probe_log_transition(p.probe_log, p.probe_cap, (uint32_t)(blockIdx.x * S + st), kSlotConsumed, kSlotEmpty);
        __syncwarp();
      }
    }
    if (lane == 0 && pk == 0) SALR_TRACE(2);
  } else if (warp == kWarpPub) {
    // ================= publisher: releases the first split partial at GPU
    // scope (fence + ticket) so the epilogue warps never stall on it
    if (early_split) {
      named_bar_sync(5, 160);  // epilogue: partial stored (bar.arrive)
      if (lane == 0) {
        const int tb = u_begin - u_begin % p.n_kt;
        fence_acq_rel_gpu();  // release (barrier + cumulativity)
        const uint32_t old = atomicAdd(&p.tickets[(tb / tiles_per_mc) * p.n_nt + (tb / p.n_kt) % p.n_nt], 1u);
        const int np = cta_of(tb + p.n_kt - 1, p.units, G) - cta_of(tb, p.units, G) + 1;
        if (!p.coop && old + 1 == (uint32_t)np) fence_acq_rel_gpu();  // we reduce it: acquire
        *early_old_slot = old;
      }
      __syncwarp();
      named_bar_arrive(6, 160);
    }
    if (p.coop && !p.cluster && u_begin < u_end) {
      // the CTA's last split partial (coop path): same release + ticket
      const int t0 = u_begin - u_begin % p.n_kt, t1 = (u_end - 1) - (u_end - 1) % p.n_kt;
      int nsp = 0, tlast = 0;
      if (!(t0 >= u_begin && t0 + p.n_kt <= u_end)) { ++nsp; tlast = t0; }
      if (t1 != t0 && !(t1 >= u_begin && t1 + p.n_kt <= u_end)) { ++nsp; tlast = t1; }
      if (nsp > (early_split ? 1 : 0)) {
        named_bar_sync(8, 160);  // epilogue: partial stored (bar.arrive)
        if (lane == 0) {
          fence_acq_rel_gpu();  // release (barrier + cumulativity)
          atomicAdd(&p.tickets[(tlast / tiles_per_mc) * p.n_nt + (tlast / p.n_kt) % p.n_nt], 1u);
        }
        __syncwarp();
      }
    }
    if (p.u_mode == 1) {
      // epoch ticket: the last CTA to finish with U advances the epoch (flips
      // the U parity) for the next launch on this workspace
      named_bar_sync(7, 160);
      if (lane == 0) {
        fence_acq_rel_gpu();
        const uint32_t d = atomicAdd(p.ctrl + kCtrlDone, 1u);
        if (d + 1 == (uint32_t)G) {
          p.ctrl[kCtrlDone] = 0u;
          fence_acq_rel_gpu();
          p.ctrl[kCtrlEpoch] = p.ctrl[kCtrlEpoch] + 1u;
        }
      }
      __syncwarp();
    }
  } else if (warp == kWarpMma) {
    // ================= MMA issuer: the whole warp walks the schedule (warp-
    // uniform state, uniform registers); one elected lane issues.  This
    // loop is the per-unit serial path of the CTA (it shares its SM
    // sub-partition with four decoder warps), so per-stage addresses advance
    // incrementally and each k-tile is one asm block.
    const uint64_t bdesc0 = desc_kmajor_sw128(smem_u32(xbuf));
    const uint32_t lo0 = (uint32_t)bdesc0, bhi = (uint32_t)(bdesc0 >> 32);
    constexpr uint32_t kLoStep = (uint32_t)(BM * 128) >> 4;  // one X stage, 16-byte units
    // The CTA owns all 512 TMEM columns, so the allocation starts at column
    // 0 (checked at setup): a compile-time base keeps the MMA operands in
    // uniform registers.
    constexpr uint32_t kTm = 0u;
    const uint32_t atm0 = kTm + a_col0, dec0 = smem_u32(decoded), emp0 = smem_u32(empty);
    int s = 0, seg = 0;
    uint32_t ph = 0, ad_ph = 0;
    int u = u_begin;
    while (u < u_end) {
      const int tile_base = u - u % p.n_kt;
      const int seg_end = min(u_end, tile_base + p.n_kt);
      const int b = NACC == 2 ? (seg & 1) : 0;
      const uint32_t acc_ph = (uint32_t)((NACC == 2 ? seg >> 1 : seg) & 1);
      const uint32_t acc = kTm + (uint32_t)(b * ACOLS);
      mbar_wait(&acc_empty[b], acc_ph ^ 1);
      tc_fence_after();
      if (S == 8 && !(p.dbg & 24) && !kProbe) {
        // Ring of 8: the stage index is a compile-time constant in each case
        // (Duff-style entry at the current stage), so barrier, TMEM and
        // descriptor offsets are immediates and the per-unit loop is two
        // barrier waits, a fence and one asm block.
        int v = u;
#define SALR_MMA_UNIT(K)                                                                              \
  case K:                                                                                             \
    if (v >= seg_end) break;                                                                          \
    mbar_wait_addr(dec0 + 8u * (K), ph);                                                              \
    tc_fence_after();                                                                                 \
    SALR_TRACE_UNIT(6, v - u_begin);                                                                  \
    mma_ktile_ts_imm<kTm + a_col0 + 32u * (K)>(acc, lo0 + (K) * kLoStep, bhi, IDESC, v != u ? 1u : 0u, \
                                                emp0 + 8u * (K));                                    \
    SALR_TRACE_UNIT(5, v - u_begin);                                                                  \
    ++v;
        while (v < seg_end) {
          switch (s) {
            SALR_MMA_UNIT(0)
            SALR_MMA_UNIT(1)
            SALR_MMA_UNIT(2)
            SALR_MMA_UNIT(3)
            SALR_MMA_UNIT(4)
            SALR_MMA_UNIT(5)
            SALR_MMA_UNIT(6)
            SALR_MMA_UNIT(7)
          }
          if (v >= seg_end) break;
          s = 0;
          ph ^= 1u;
        }
#undef SALR_MMA_UNIT
        // stage and phase of the next unit
        s = (seg_end - u_begin) % 8;
        ph = (uint32_t)(((seg_end - u_begin) / 8) & 1);
      } else {
      int sg = s;
      uint32_t lo = lo0 + (uint32_t)sg * kLoStep, atm = atm0 + 32u * (uint32_t)sg;
      uint32_t dad = dec0 + 8u * (uint32_t)sg, ead = emp0 + 8u * (uint32_t)sg;
      for (int v = u; v < seg_end; ++v) {
        mbar_wait_addr(dad, ph);  // decoded tile and X tile
        if (kProbe) {
          if (lane == 0)
            probe_log_transition(p.probe_log, p.probe_cap, (uint32_t)(blockIdx.x * S + sg), kSlotFilled,
                                 kSlotConsumed);
          probe_jitter(p.probe_ns, p.probe_seed ^ 0x5bd1e995u, (uint32_t)v, 1u);
          __syncwarp();
        }
        tc_fence_after();
        SALR_TRACE_UNIT(6, v - u_begin);
        if (p.dbg & 8) {  // experiment: commit without MMAs (wrong results)
          if (elect_one()) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(ead) : "memory");
          __syncwarp();
        } else {
          mma_ktile_ts(acc, atm, lo, bhi, IDESC, v != u ? 1u : 0u, ead);
        }
        SALR_TRACE_UNIT(5, v - u_begin);
        if (++sg == S) {
          sg = 0;
          ph ^= 1u;
          lo = lo0;
          atm = atm0;
          dad = dec0;
          ead = emp0;
        } else {
          lo += kLoStep;
          atm += 32u;
          dad += 8u;
          ead += 8u;
        }
      }
      s = sg;
      }
      if (u == tile_base && p.ra) {
        mbar_wait(ad_full, ad_ph);
        ad_ph ^= 1;
        tc_fence_after();
        if (elect_one()) {
          for (int a = 0; a < p.ra; ++a) {
            uint8_t* blk = adbuf + (size_t)a * (kAdTileBytes + 2u * BM * 128u);
            const uint64_t adesc = desc_kmajor_sw128(smem_u32(blk));
            const uint64_t hdesc = desc_kmajor_sw128(smem_u32(blk + kAdTileBytes));
            const uint64_t ldesc = desc_kmajor_sw128(smem_u32(blk + kAdTileBytes + BM * 128));
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_ss(acc, adesc + 2 * j, hdesc + 2 * j, IDESC, 1u);
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_ss(acc, adesc + 2 * j, ldesc + 2 * j, IDESC, 1u);
          }
          tc_commit(ad_empty);
        }
        __syncwarp();
      }
      if (elect_one()) {
        tc_commit(&acc_full[b]);
        SALR_TRACE(6);
      }
      __syncwarp();
      ++seg;
      u = seg_end;
    }
  } else if (warp >= kFirstDecWarp && warp < kFirstEpiWarp) {
    // ================= decoders (TB2 records).  Group g = units it = g (mod
    // kDecGroups); warp (g, part, q) owns TMEM lanes 32q..32q+31 (output
    // columns of group q) and bands part*BPW .. of the tile.  Per lane (one
    // output column) and 4-row band the values are contiguous: the band's
    // run start is bandoff[q][b] + (exclusive warp prefix of the band
    // counts), and a predicated pointer chain expands the 4 rows -- no
    // per-element rank popcounts.
    constexpr int BPW = RPW / 4;  // bands per decoder warp
    const int dw = warp - kFirstDecWarp;
    const int grp = dw / WPG;
    const int part = (dw % WPG) >> 2;
    const int q = warp & 3;
    const uint32_t lane_tm = (uint32_t)(32 * q) << 16;
    int s = grp;  // S is a multiple of kDecGroups (host)
    uint32_t ph = 0;
    for (int it = u_begin + grp; it < u_end; it += kDecGroups) {
      mbar_wait(&full[s], ph);
      if (lane == 0 && (dw % WPG) == 0) SALR_TRACE_UNIT(1, it - u_begin);
      if (kProbe) {
        if (lane == 0 && (dw % WPG) == 0)
          probe_log_transition(p.probe_log, p.probe_cap, (uint32_t)(blockIdx.x * S + s), kSlotEmpty, kSlotFilled);
        probe_jitter(p.probe_ns, p.probe_seed, (uint32_t)it, (uint32_t)warp);
        __syncwarp();
      }
      const uint8_t* rec = recbuf + (size_t)s * p.rec_slot;
      const uint32_t taddr = tmem + lane_tm + a_col0 + 32u * s + (uint32_t)(2 * BPW * part);
      if (!(p.dbg & 1)) {
        if (p.nm24)
          decode_tile_nm24<BPW>(smem_u32(rec), taddr, q, lane, part);
        else
          decode_tile_tb2<BPW>(smem_u32(rec), taddr, q, lane, lut_s, part);
        if (lane == 0 && (dw % WPG) == 0) SALR_TRACE_UNIT(11, it - u_begin);
        tc_wait_st();
        if (lane == 0 && (dw % WPG) == 0) SALR_TRACE_UNIT(13, it - u_begin);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&decoded[s]);
        if (dw == 0) SALR_TRACE(it == u_begin ? 4 : 11);
        if ((dw % WPG) == 0) SALR_TRACE_UNIT(3, it - u_begin);
        if ((dw % WPG) == WPG - 1) SALR_TRACE_UNIT(4, it - u_begin);
      }
      s += kDecGroups;
      if (s >= S) { s -= S; ph ^= 1; }
    }
  } else if (warp >= kFirstEpiWarp && warp < kFirstEpiWarp + 4) {
    // ================= epilogue
    const int q = warp & 3;
    const uint32_t lane_tm = (uint32_t)(32 * q) << 16;
    const int etid = (warp - kFirstEpiWarp) * 32 + (int)lane;  // 0..127
    const int rp = 64 * p.ra;
    uint32_t par = 0;
    if (p.u_mode == 1) par = *reinterpret_cast<volatile uint32_t*>(p.ctrl + kCtrlEpoch) & 1u;
    bool u_ok = false;
    uint32_t ad_ph = 0;
    // adapter operands of the output tile whose first k-unit is useg (a
    // first-k segment) into the single adapter slot: B_cat^T tile by TMA,
    // U hi/lo (BM x 64 per rank block, K-major, 128B swizzle) built from the
    // fixed-point U or loaded by TMA.  Prepared as early as the slot allows
    // (the MMA only needs it after that segment's k-loop).
    auto prep_adapter = [&](int useg) {
      const int nt = (useg / p.n_kt) % p.n_nt;
      const int mc = useg / (p.n_kt * p.n_nt);
      // ---- adapter operands of this output tile into the adapter slot:
      // B_cat^T tile by TMA, U hi/lo (BM x 64 per rank block, K-major, 128B
      // swizzle) built from the fixed-point U or loaded by TMA.
      if (etid == 0) {
        mbar_wait(ad_empty, ad_ph ^ 1);
        // the B_cat^T tile does not depend on U: start its fetch now (the
        // transaction bytes are expected below, with the single arrive)
        for (int a = 0; a < p.ra; ++a)
          tma_2d_g2s(adbuf + (size_t)a * (kAdTileBytes + 2u * BM * 128u), &bmap, 64 * a, nt * kTileN, ad_full);
      }
      named_bar_sync(1, 128);
      if (p.u_mode == 1) {
        if (!u_ok) {
          if (etid == 0) {
            // acquire pairs with the producers' fence + counter increment
            while (ld_acquire_u32(p.ctrl + kCtrlReady + par) < (uint32_t)((p.K + kUSlice - 1) / kUSlice))
              __nanosleep(32);
            SALR_TRACE(14);
          }
          named_bar_sync(1, 128);
          u_ok = true;
        }
        const unsigned long long* uacc = p.u_acc + (size_t)par * kUAccElems;
        for (int e = etid; e < BM * 32 * p.ra; e += 128) {  // (m, r pair) items
          const int a = e / (BM * 32);
          const int m = (e / 32) % BM;
          const int rr = 2 * (e % 32);  // r within the 64-block
          const int gm = mc * BM + m;
          float u0 = 0.f, u1 = 0.f;
          if (gm < p.M) {
            const unsigned long long* src = uacc + (size_t)gm * rp + 64 * a + rr;
            u0 = (float)((double)(long long)__ldcg(src) * (1.0 / (double)(1ll << kUFrac)));
            u1 = (float)((double)(long long)__ldcg(src + 1) * (1.0 / (double)(1ll << kUFrac)));
          }
          const __nv_bfloat16 h0 = __float2bfloat16_rn(u0), h1 = __float2bfloat16_rn(u1);
          const __nv_bfloat16 l0 = __float2bfloat16_rn(u0 - __bfloat162float(h0));
          const __nv_bfloat16 l1 = __float2bfloat16_rn(u1 - __bfloat162float(h1));
          const uint32_t boff = (uint32_t)(m * 128 + (((rr >> 3) ^ (m & 7)) << 4) + 2 * (rr & 7));
          uint8_t* blk = adbuf + (size_t)a * (kAdTileBytes + 2u * BM * 128u);
          *reinterpret_cast<__nv_bfloat162*>(blk + kAdTileBytes + boff) = __halves2bfloat162(h0, h1);
          *reinterpret_cast<__nv_bfloat162*>(blk + kAdTileBytes + BM * 128 + boff) = __halves2bfloat162(l0, l1);
        }
        fence_proxy_async_smem();
      }
      named_bar_sync(1, 128);
      if (etid == 0) {
        if (p.u_mode == 2 && !u_ok) {
          pdl_wait();  // U hi/lo come from the preceding kernel
          u_ok = true;
        }
        const uint32_t ubytes = p.u_mode == 2 ? 2u * BM * 128u : 0u;
        mbar_arrive_expect_tx(ad_full, (uint32_t)p.ra * (kAdTileBytes + ubytes));
        for (int a = 0; a < p.ra; ++a) {
          uint8_t* blk = adbuf + (size_t)a * (kAdTileBytes + 2u * BM * 128u);
          if (p.u_mode == 2) {
            tma_2d_g2s(blk + kAdTileBytes, &uhimap, 64 * a, mc * BM, ad_full);
            tma_2d_g2s(blk + kAdTileBytes + BM * 128, &ulomap, 64 * a, mc * BM, ad_full);
          }
        }
      }
      ad_ph ^= 1;
    };
    auto next_first_k = [&](int from) {  // first tile boundary >= from within the range
      const int t = from % p.n_kt == 0 ? from : from - from % p.n_kt + p.n_kt;
      return t < u_end ? t : u_end;
    };
    int next_ad = p.ra ? next_first_k(u_begin) : u_end;
    if (next_ad < u_end) {
      prep_adapter(next_ad);
      next_ad = next_first_k(next_ad + 1);
    }
    // Sum the partial tiles of a split output tile (the unit range starting
    // at tile_base) over CTAs c_first..c_last in that fixed order
    // (deterministic); this CTA takes share `share` of `nshare` row slices.
    auto reduce_split = [&](int tile_base, int share, int nshare, bool reset, int t0, int nthr) {
      const int nt = (tile_base / p.n_kt) % p.n_nt;
      const int mc = tile_base / (p.n_kt * p.n_nt);
      const int rows = min(BM, p.M - mc * BM);
      const int c_first = cta_of(tile_base, p.units, G), c_last = cta_of(tile_base + p.n_kt - 1, p.units, G);
      // CTA c > c_first begins inside this tile (its slot 0); c_first
      // holds it in slot 1 unless its range starts exactly at the tile.
      const int cb_first = (int)((int64_t)c_first * p.units / G);
      const size_t tile_elems = (size_t)BM * kTileN;
      const float* p_first = p.partials + ((size_t)c_first * 2 + (cb_first >= tile_base ? 0 : 1)) * tile_elems;
      const int r0 = share * rows / nshare, r1 = (share + 1) * rows / nshare;
      auto store_y = [&](size_t o, int col, float v) {
        if (col >= p.N) return;
        if (p.y_dtype == kF32) static_cast<float*>(p.y)[o] = v;
        else static_cast<__nv_bfloat16*>(p.y)[o] = __float2bfloat16_rn(v);
      };
      if (r1 - r0 <= 2) {
        // few rows (decode-size M): one element per thread and pass, up to
        // 16 partials in flight -- a single round trip for most tiles
        for (int e = etid - t0; e < (r1 - r0) * kTileN; e += nthr) {
          const int m = r0 + e / kTileN, cl = e % kTileN;
          const size_t off = (size_t)m * kTileN + cl;
          float acc = __ldcg(p_first + off);
          for (int c = c_first + 1; c <= c_last; c += 8) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + i <= c_last) v[i] = __ldcg(p.partials + (size_t)(c + i) * 2 * tile_elems + off);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + i <= c_last) acc += v[i];
          }
          store_y((size_t)(mc * BM + m) * p.ldy + nt * kTileN + cl, nt * kTileN + cl, acc);
        }
      } else if (c_last - c_first <= 1) {
        // two partials (large shapes: tiles split over 2 CTAs), many chunks
        // per thread: 4-column chunks, kIPT per thread per pass, every
        // partial of the pass loaded before any sum (one L2 round trip per
        // pass instead of one per chunk), summed in CTA order
        constexpr int kIPT = 4;
        const int items = (r1 - r0) * (kTileN / 4);
        for (int e0 = etid - t0; e0 < items; e0 += nthr * kIPT) {
          float4 acc[kIPT];
          size_t offs[kIPT];
#pragma unroll
          for (int i = 0; i < kIPT; ++i) {
            const int e = e0 + i * nthr;
            const int m = r0 + e / (kTileN / 4), c4 = 4 * (e % (kTileN / 4));
            offs[i] = (size_t)m * kTileN + c4;
            if (e < items) acc[i] = __ldcg(reinterpret_cast<const float4*>(p_first + offs[i]));
          }
          for (int c = c_first + 1; c <= c_last; c += 2) {
            float4 v[2][kIPT];
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int i = 0; i < kIPT; ++i)
                if (c + j <= c_last && e0 + i * nthr < items)
                  v[j][i] = __ldcg(reinterpret_cast<const float4*>(p.partials + (size_t)(c + j) * 2 * tile_elems +
                                                                   offs[i]));
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int i = 0; i < kIPT; ++i)
                if (c + j <= c_last && e0 + i * nthr < items) {
                  acc[i].x += v[j][i].x;
                  acc[i].y += v[j][i].y;
                  acc[i].z += v[j][i].z;
                  acc[i].w += v[j][i].w;
                }
          }
#pragma unroll
          for (int i = 0; i < kIPT; ++i) {
            const int e = e0 + i * nthr;
            if (e >= items) continue;
            const int m = r0 + e / (kTileN / 4), c4 = 4 * (e % (kTileN / 4));
            const size_t o = (size_t)(mc * BM + m) * p.ldy + nt * kTileN + c4;
            store_y(o, nt * kTileN + c4, acc[i].x);
            store_y(o + 1, nt * kTileN + c4 + 1, acc[i].y);
            store_y(o + 2, nt * kTileN + c4 + 2, acc[i].z);
            store_y(o + 3, nt * kTileN + c4 + 3, acc[i].w);
          }
        }
      } else {
        // one 4-column chunk per thread and pass; the partials of a chunk are
        // loaded in batches of 8 independent 16-byte loads
        for (int e = etid - t0; e < (r1 - r0) * (kTileN / 4); e += nthr) {
          const int m = r0 + e / (kTileN / 4), c4 = 4 * (e % (kTileN / 4));
          const size_t off = (size_t)m * kTileN + c4;
          float4 acc = __ldcg(reinterpret_cast<const float4*>(p_first + off));
          for (int c = c_first + 1; c <= c_last; c += 8) {
            float4 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + i <= c_last)
                v[i] = __ldcg(reinterpret_cast<const float4*>(p.partials + (size_t)(c + i) * 2 * tile_elems + off));
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c + i <= c_last) {
                acc.x += v[i].x;
                acc.y += v[i].y;
                acc.z += v[i].z;
                acc.w += v[i].w;
              }
          }
          const size_t o = (size_t)(mc * BM + m) * p.ldy + nt * kTileN + c4;
          store_y(o, nt * kTileN + c4, acc.x);
          store_y(o + 1, nt * kTileN + c4 + 1, acc.y);
          store_y(o + 2, nt * kTileN + c4 + 2, acc.z);
          store_y(o + 3, nt * kTileN + c4 + 3, acc.w);
        }
      }
      if (reset && etid == t0) p.tickets[mc * p.n_nt + nt] = 0u;
    };
    auto tile_np = [&](int tb) {
      return cta_of(tb + p.n_kt - 1, p.units, G) - cta_of(tb, p.units, G) + 1;
    };
    auto tile_ticket = [&](int tb) {
      return &p.tickets[(tb / (p.n_kt * p.n_nt)) * p.n_nt + (tb / p.n_kt) % p.n_nt];
    };
    bool early_pub = false;  // first split segment already published in the loop
    int seg = 0;
    int u = u_begin;
    while (u < u_end) {
      const int tile_base = u - u % p.n_kt;
      const int seg_end = min(u_end, tile_base + p.n_kt);
      const bool full_cover = (u == tile_base) && (seg_end == tile_base + p.n_kt);
      const int nt = (u / p.n_kt) % p.n_nt;
      const int mc = u / (p.n_kt * p.n_nt);
      const int b = NACC == 2 ? (seg & 1) : 0;
      const uint32_t acc_ph = (uint32_t)((NACC == 2 ? seg >> 1 : seg) & 1);
      // long wait: try_wait suspends the warp in hardware (no issue slots)
      // and wakes it as soon as the phase completes
      mbar_wait(&acc_full[b], acc_ph);
      tc_fence_after();
      if (etid == 0 && seg == 0) SALR_TRACE(7);
      // partial slot of this CTA: 0 for its first segment, 1 otherwise
      float* part_tile = p.partials + ((size_t)blockIdx.x * 2 + (u == u_begin ? 0 : 1)) * (size_t)BM * kTileN;
      const int nl = 32 * q + (int)lane;
      const int n = nt * kTileN + nl;
      const bool n_ok = n < p.N;
      const int rows = min(BM, p.M - mc * BM);
      if (etid == 0) SALR_TRACE_UNIT(12, seg);
      // Drain the accumulator 16 rows at a time (two loads in flight).  The
      // destination mode is uniform per segment, so each mode gets its own
      // branch-free store loop:
      //   full tile      -> y (row-major, lanes along n: coalesced)
      //   cluster split  -> own smem, n-major [128][BM+4] (16-byte stores,
      //                     conflict-free), reduced through DSMEM at the end
      //   global split   -> partial slot [BM][128] (coalesced)
      const int mode = full_cover ? (p.y_dtype == kF32 ? 0 : 1) : (p.cluster ? 2 : 3);
      float* const sp_col = reinterpret_cast<float*>(xbuf) + nl * (BM + 4);
      const size_t yrow0 = (size_t)(mc * BM) * p.ldy + n;
#pragma unroll 1
      for (int c0 = 0; c0 < rows; c0 += 8) {
        uint32_t r[8];
        SALR_TMEM_LD_X8(tmem + lane_tm + (uint32_t)(b * ACOLS + c0), r);
        tc_wait_ld();
        if (mode == 2) {
          *reinterpret_cast<uint4*>(sp_col + c0) = make_uint4(r[0], r[1], r[2], r[3]);
          *reinterpret_cast<uint4*>(sp_col + c0 + 4) = make_uint4(r[4], r[5], r[6], r[7]);
        } else if (mode == 3) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (c0 + i < rows) __stcg(part_tile + (size_t)(c0 + i) * kTileN + nl, __uint_as_float(r[i]));
        } else if (n_ok) {
          if (mode == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c0 + i < rows) static_cast<float*>(p.y)[yrow0 + (size_t)(c0 + i) * p.ldy] = __uint_as_float(r[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c0 + i < rows)
                static_cast<__nv_bfloat16*>(p.y)[yrow0 + (size_t)(c0 + i) * p.ldy] =
                    __float2bfloat16_rn(__uint_as_float(r[i]));
          }
        }
      }
      if (etid == 0 && seg == 0) SALR_TRACE(25);
      if (etid == 0) SALR_TRACE_UNIT(14, seg);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      // this segment's adapter (if any) was consumed before acc_full: the
      // slot is free for the next first-k segment
      if (next_ad < u_end && u == tile_base) {
        prep_adapter(next_ad);
        next_ad = next_first_k(next_ad + 1);
      }
      if (!full_cover && !p.cluster && seg_end < u_end) {
        // (== early_split: only the first segment can be split and followed)
        // a split segment with more work behind it (only the CTA's first
        // segment can be one): publish its partial now, off the critical
        // path.  (Its last-CTA reduction, if ours -- rare: the CTA before us
        // finishes its part of this tile last -- waits for the tail below.)
        named_bar_arrive(5, 160);  // hand the stored partial to the publisher warp
        early_pub = true;
      }

      ++seg;
      u = seg_end;
    }
    // ---- split-K tail (global path).  A CTA shares at most two output tiles
    // (its first and its last segment).  The first was published in the loop
    // if work followed it; publish the rest with one release and relaxed
    // ticket increments issued back to back (round trips overlap), then
    //   coop (M >= 16): wait for every participant, reduce our row share, or
    //   last-CTA:       the CTA completing a ticket reduces the whole tile.
    // The in-kernel U epoch ticket rides along: this CTA is done with U.
    int tl[2];
    int nsplit = 0;
    if (!p.cluster && u_begin < u_end) {
      const int t0 = u_begin - u_begin % p.n_kt, t1 = (u_end - 1) - (u_end - 1) % p.n_kt;
      if (!(t0 >= u_begin && t0 + p.n_kt <= u_end)) tl[nsplit++] = t0;
      if (t1 != t0 && !(t1 >= u_begin && t1 + p.n_kt <= u_end)) tl[nsplit++] = t1;
    }
    // tiles still to publish: all but the early-published first one
    const int jpub = early_pub ? 1 : 0;
    if (nsplit > jpub) named_bar_sync(1, 128);  // every partial of this CTA stored (CTA scope)
    if (early_pub) named_bar_sync(6, 160);  // the publisher's ticket value is in
    // this CTA is done with U: the publisher warp takes the epoch ticket
    // off the epilogue's critical path
    // coop: the publisher warp releases the last partial too (nobody here
    // needs the ticket's old value)
    if (p.coop && nsplit > jpub) named_bar_arrive(8, 160);
    if (p.u_mode == 1) named_bar_arrive(7, 160);
    if (etid == 0 && nsplit && !p.coop) {
      SALR_TRACE(29);
      uint32_t old[2] = {early_pub ? *early_old_slot : 0u, 0u};
      // acq_rel: publishes the last partial and acquires the others'
      if (nsplit > jpub) old[nsplit - 1] = ticket_add_acq_rel(tile_ticket(tl[nsplit - 1]), 1u);
      uint32_t lf = 0;
#pragma unroll
      for (int j = 0; j < nsplit; ++j)
        if (!p.coop && old[j] + 1 == (uint32_t)tile_np(tl[j])) lf |= 1u << j;
      *last_flag = lf;
      SALR_TRACE(30);
    }
    if (nsplit) {
      named_bar_sync(1, 128);
      if (p.coop) {
        // wait for every participant of a tile, reduce our row share
#pragma unroll
        for (int j = 0; j < nsplit; ++j) {
          const int tb = tl[j], np = tile_np(tb);
          uint32_t* tk = tile_ticket(tb);
          if (etid == 0)
            while (ld_acquire_u32(tk) < (uint32_t)np) __nanosleep(32);
          named_bar_sync(1, 128);
          reduce_split(tb, (int)blockIdx.x - cta_of(tb, p.units, G), np, false, 0, 128);
          named_bar_sync(1, 128);
          if (etid == 0) {
            SALR_TRACE(22);
            // the last participant out resets both counters for the next launch
            if (atomicAdd(tk + kDoneTicketOff, 1u) + 1 == (uint32_t)np) {
              tk[0] = 0u;
              tk[kDoneTicketOff] = 0u;
            }
          }
        }
      } else {
        const uint32_t lf = *last_flag;
#pragma unroll
        for (int j = 0; j < nsplit; ++j)
          if ((lf >> j) & 1u) reduce_split(tl[j], 0, 1, true, 0, 128);
        if (etid == 0 && lf) SALR_TRACE(31);
      }
    }
    if (etid == 0) SALR_TRACE(8);
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) SALR_TRACE(26);
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (p.cluster) {
    // split-K reduction of this cluster's output tile through distributed
    // shared memory: CTA rank j sums rows [j, j+1) * rows / np of the np
    // partials in rank (= k) order -- the same order as the global path.
    cluster_sync_all();  // every partial of the cluster is in shared memory
    if (threadIdx.x == 0) SALR_TRACE(27);
    const int np = p.cluster;
    const int rank = (int)(blockIdx.x % (unsigned)np);
    const int tb = u_begin - u_begin % p.n_kt;
    const int nt = (tb / p.n_kt) % p.n_nt, mc = tb / (p.n_kt * p.n_nt);
    const int rows = min(BM, p.M - mc * BM);
    // groups of 4 rows: CTA rank j owns groups [j, j+1) * ng / np
    const int ng = (rows + 3) / 4;
    const int g0 = rank * ng / np, g1 = (rank + 1) * ng / np;
    const uint32_t sp = smem_u32(xbuf);
    for (int e = threadIdx.x; e < (g1 - g0) * kTileN; e += threads_for(BM)) {
      const int nl = e % kTileN, m = 4 * (g0 + e / kTileN);
      const uint32_t a = sp + (uint32_t)((nl * (BM + 4) + m) * 4);
      // every remote load in flight before the (rank-ordered) sums
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < np) v[j] = ld_dsmem_f4(a, (uint32_t)j);
      float4 acc = v[0];
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (j < np) {
          acc.x += v[j].x;
          acc.y += v[j].y;
          acc.z += v[j].z;
          acc.w += v[j].w;
        }
      const int n = nt * kTileN + nl;
      if (n < p.N) {
        const float o4[4] = {acc.x, acc.y, acc.z, acc.w};
        const size_t o = (size_t)(mc * BM + m) * p.ldy + n;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (m + i >= rows) break;
          if (p.y_dtype == kF32) static_cast<float*>(p.y)[o + (size_t)i * p.ldy] = o4[i];
          else static_cast<__nv_bfloat16*>(p.y)[o + (size_t)i * p.ldy] = __float2bfloat16_rn(o4[i]);
        }
      }
    }
    if (threadIdx.x == 0) SALR_TRACE(28);
    cluster_sync_all();  // no CTA leaves while its partial is being read
  }
  if (threadIdx.x == 0) SALR_TRACE(9);
}

// U[m, r] = sum_k X[m, k] * A_cat[k, r] (fp32), written as bf16 hi + lo
// halves (U = hi + lo to ~2^-16 relative).  Grid (m-blocks of 8 rows, K
// splits, r blocks of 64); every block stores its partial, and the last block
// of each (m-block, r-block) -- found with a self-resetting ticket -- sums
// the K-split partials in split order, so U is bit-reproducible.
__global__ void __launch_bounds__(256) adapter_u_kernel(const __nv_bfloat16* __restrict__ x, int64_t M, int64_t K,
                                                        int64_t ldx, const __nv_bfloat16* __restrict__ acat,
                                                        int r_pad, int64_t kchunk, float* __restrict__ u_part,
                                                        uint32_t* __restrict__ u_tickets,
                                                        __nv_bfloat16* __restrict__ u_hi,
                                                        __nv_bfloat16* __restrict__ u_lo) {
  pdl_launch_dependents();
  constexpr int MB = 8;
  __shared__ uint32_t is_last;
  const int r = threadIdx.x + 64 * blockIdx.z;
  const int ty = threadIdx.y;
  const int64_t m0 = (int64_t)blockIdx.x * MB;
  const int64_t k0 = (int64_t)blockIdx.y * kchunk;
  const int64_t k1 = min(K, k0 + kchunk);
  float acc0 = 0.f, acc1 = 0.f;
  const int64_t ma = m0 + ty, mb = m0 + ty + 4;
  const bool va = ma < M, vb = mb < M;
  const __nv_bfloat16* xa = x + (va ? ma : 0) * ldx;
  const __nv_bfloat16* xb = x + (vb ? mb : 0) * ldx;
  const int kn = (int)(k1 - k0);
  const __nv_bfloat16* ap = acat + k0 * r_pad + r;
  int k = 0;
  for (; k + 8 <= kn; k += 8) {  // 24 independent loads in flight per thread
    float a[8], fa[8], fb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __bfloat162float(ap[(k + i) * r_pad]);
      fa[i] = __bfloat162float(xa[k0 + k + i]);
      fb[i] = __bfloat162float(xb[k0 + k + i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc0 = fmaf(fa[i], a[i], acc0);
      acc1 = fmaf(fb[i], a[i], acc1);
    }
  }
  for (; k < kn; ++k) {
    const float a = __bfloat162float(ap[k * r_pad]);
    acc0 = fmaf(__bfloat162float(xa[k0 + k]), a, acc0);
    acc1 = fmaf(__bfloat162float(xb[k0 + k]), a, acc1);
  }
  float* part = u_part + (size_t)blockIdx.y * M * r_pad;
  if (va) __stcg(part + ma * r_pad + r, acc0);
  if (vb) __stcg(part + mb * r_pad + r, acc1);
  fence_acq_rel_gpu();
  __syncthreads();
  uint32_t* ticket = u_tickets + (size_t)blockIdx.x * gridDim.z + blockIdx.z;
  if (threadIdx.x == 0 && ty == 0) is_last = (atomicAdd(ticket, 1u) + 1 == gridDim.y) ? 1u : 0u;
  __syncthreads();
  if (!is_last) return;
  fence_acq_rel_gpu();
  for (int j = 0; j < 2; ++j) {
    const int64_t m = j ? mb : ma;
    if (m >= M) continue;
    float sum = 0.f;
    for (unsigned ks = 0; ks < gridDim.y; ++ks) sum += __ldcg(u_part + (size_t)ks * M * r_pad + m * r_pad + r);
    const __nv_bfloat16 h = __float2bfloat16_rn(sum);
    u_hi[m * r_pad + r] = h;
    u_lo[m * r_pad + r] = __float2bfloat16_rn(sum - __bfloat162float(h));
  }
  if (threadIdx.x == 0 && ty == 0) *ticket = 0u;
}

// --------------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Experiment switches (environment) exist only in debug builds
// (-DSALR_DEBUG): a release library never changes its schedule or skips work
// because of the environment.
static const char* dbg_env(const char* name) {
#ifdef SALR_DEBUG
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Host-side caches are per device ordinal: function attributes, SM counts
// and occupancy answers belong to one device context.
constexpr int kMaxDevices = 64;
static int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    (void)cudaGetLastError();
    dev = 0;
  }
  return dev;
}
static int sm_count() {
  static int n[kMaxDevices] = {};
  const int dev = cur_device();
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// bf16 2-D tensor map over a row-major (rows x cols) matrix, box (64 cols, box_rows), 128B swizzle.
static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld_elems,
                    int box_rows) {
  EncodeTiledFn enc = get_encode_tiled();
  SALR_CHECK_ARG(enc != nullptr, SALR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
  const cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SALR_CHECK_ARG(cr == CUDA_SUCCESS, SALR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  return SALR_OK;
}

#include "salr_prefill.cuh"
#include "salr_chain.cuh"

static unsigned long long* g_trace = nullptr;  // set by salr_debug_set_trace (tools only)
static uint32_t* g_probe_log = nullptr;         // set by salr_debug_set_probe (tests / tools)
static uint32_t g_probe_cap = 0, g_probe_ns = 0, g_probe_seed = 0;

static int pick_bm(int64_t M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  return 128;
}

// deepest ring that fits shared memory and TMEM
// Deepest ring that fits shared memory and TMEM (slots sized for the largest
// record of the matrix: ~9.6 KB at 50% sparsity instead of the 17.4 KB worst
// case).
static int max_stages(int bm, int ra, uint32_t rec_slot, int cap) {
  const int acc = nacc_for(bm) * acc_cols_for(bm);
  const int tmem_stages = (512 - ((acc + 31) & ~31)) / 32;
  // default cap 8 slots (measured: 12 are ~1-2 % slower on every Llama
  // shape, 4 are 15 % slower); an explicit request may go deeper
  int s = cap;
  if (s > tmem_stages) s = tmem_stages;
  while (s > 1 && smem_plan(bm, s, ra, rec_slot).total > kSmemMaxLinear) --s;
  if (s > 4) s &= ~3;  // a multiple of the decoder group count
  return s;
}

// configuration of the most recent linear launch (salr_debug_last_launch)
static int g_last_launch[12] = {};

template <int BM, int NG, bool kProbe = false>
static int launch_linear_g(const CUtensorMap* maps, LinearParams p, int ctas, cudaStream_t s, bool pdl) {
  auto kern = salr_linear_kernel<BM, NG, kProbe>;
  const SmemPlan plan = smem_plan(BM, p.stages, p.ra, p.rec_slot);
  p.x_off = plan.x_off;
  p.rec_off = plan.rec_off;
  p.base_off = plan.base_off;
  p.ad_off = plan.ad_off;
  p.bar_off = plan.bar_off;
  const int dev = cur_device();
  static bool attr_done[kMaxDevices] = {};
  if (!attr_done[dev]) {
    SALR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxLinear));
    attr_done[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(threads_for(BM));
  cfg.dynamicSmemBytes = plan.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (p.cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)p.cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = (unsigned)na;
  const int cluster_req = p.cluster;
  int cluster_max = -1;
  if (p.cluster > 1) {
    // every cluster must be resident at once (else fall back to the global
    // split-K path); cached per configuration
    static int64_t cached_key[kMaxDevices], cached_max[kMaxDevices];
    static bool cached_init = false;
    if (!cached_init) {
      for (int d = 0; d < kMaxDevices; ++d) cached_key[d] = -1;
      cached_init = true;
    }
    const int64_t key = ((int64_t)p.cluster << 32) | plan.total;
    if (key != cached_key[dev]) {
      int n = 0;
      cudaLaunchConfig_t q = cfg;
      q.attrs = attr + (pdl ? 1 : 0);
      q.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess) {
        (void)cudaGetLastError();
        n = 0;
      }
      cached_key[dev] = key;
      cached_max[dev] = n;
    }
    cluster_max = (int)cached_max[dev];
    if (cached_max[dev] * p.cluster < ctas) {
      p.cluster = 0;
      cfg.numAttrs = (unsigned)(na - 1);
    }
  }
  // In-kernel U (u_mode 1) and the cooperative split-K reduction wait on
  // other CTAs of the grid: forward progress needs every CTA resident at
  // once.  A cooperative launch makes the driver guarantee that (or fail
  // the launch) instead of relying on grid <= SM count alone, so a
  // concurrent kernel (an NCCL collective on another stream, MPS) cannot
  // deadlock the spinning CTAs.  A programmatic-dependent launch (flag
  // SALR_FLAG_PDL, chained kernels of one stream) is not co-scheduled --
  // co-scheduling would wait for the preceding grid to drain and void the
  // overlap -- so it is checked against occupancy instead, and the PDL
  // contract (include/salr_b200.h) excludes concurrent kernels that wait on
  // this grid.
  int coop_launch = 0;
  if ((p.u_mode == 1 || p.coop) && pdl) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads_for(BM), plan.total) != cudaSuccess) {
      (void)cudaGetLastError();
      per_sm = 1;
    }
    SALR_CHECK_ARG((int64_t)per_sm * sm_count() >= ctas, SALR_ERR_CUDA,
                   "grid of %d CTAs cannot be co-resident (%d per SM)", ctas, per_sm);
  }
  if ((p.u_mode == 1 || p.coop) && !pdl) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeCooperative;
    attr[cfg.numAttrs].val.cooperative = 1;
    cfg.numAttrs += 1;
    coop_launch = 1;
  }
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], p);
  if (le != cudaSuccess && coop_launch) {
    // the driver refused the co-scheduled launch (attribute combination or
    // too large a grid): launch without it only if every CTA fits at once
    (void)cudaGetLastError();
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads_for(BM), plan.total) != cudaSuccess) {
      (void)cudaGetLastError();
      per_sm = 0;
    }
    SALR_CHECK_ARG((int64_t)per_sm * sm_count() >= ctas, SALR_ERR_CUDA,
                   "grid of %d CTAs cannot be co-resident (%d per SM): %s", ctas, per_sm, cudaGetErrorString(le));
    cfg.numAttrs -= 1;
    coop_launch = 0;
    le = cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], p);
  }
  SALR_CUDA_TRY(le);
  const int info[12] = {ctas, p.stages, BM, NG, p.u_mode, p.coop, p.cluster, pdl ? 1 : 0,
                        cluster_req, cluster_max, (int)plan.total, coop_launch};
  for (int i = 0; i < 12; ++i) g_last_launch[i] = info[i];
  return SALR_OK;
}

// Decoder groups: 4 by default (SALR_DEC_GROUPS overrides for experiments),
// reduced to a divisor of the ring depth (stage ownership, see the kernel).
static int dec_groups(int stages) {
  static int g = 0;
  if (!g) {
    const char* e = dbg_env("SALR_DEC_GROUPS");
#ifndef SALR_DEFAULT_DEC_GROUPS
#define SALR_DEFAULT_DEC_GROUPS 4
#endif
    g = e ? atoi(e) : SALR_DEFAULT_DEC_GROUPS;
    if (g != 1 && g != 2 && g != 4) g = 4;
  }
  int ng = g;
  while (ng > 1 && stages % ng) ng >>= 1;
  return ng;
}

template <int BM>
static int launch_linear(const CUtensorMap* maps, const LinearParams& p, int ctas, cudaStream_t s, bool pdl) {
  switch (dec_groups(p.stages)) {
    case 1: return launch_linear_g<BM, 1>(maps, p, ctas, s, pdl);
    case 2: return launch_linear_g<BM, 2>(maps, p, ctas, s, pdl);
    default: return launch_linear_g<BM, 4>(maps, p, ctas, s, pdl);
  }
}

// The probed instantiations (salr_debug_set_probe): decode-size tiles of
// BM = 16 tokens only, so the release kernels carry no probe code.
static int launch_linear_probed(const CUtensorMap* maps, const LinearParams& p, int ctas, cudaStream_t s, bool pdl) {
  switch (dec_groups(p.stages)) {
    case 1: return launch_linear_g<16, 1, true>(maps, p, ctas, s, pdl);
    case 2: return launch_linear_g<16, 2, true>(maps, p, ctas, s, pdl);
    default: return launch_linear_g<16, 4, true>(maps, p, ctas, s, pdl);
  }
}

// Prefill kernel: deepest X ring (and a 4-slot record ring) that fits.
static int launch_prefill(const CUtensorMap* maps, PrefillParams pp, cudaStream_t s, bool pdl) {
  pp.SR = 6;
  pp.SX = 12;
  while (pp.SX > 2 && pf_plan(pp.SR, pp.SX, pp.ra, pp.rec_slot).total > kSmemMax) --pp.SX;
  const PfPlan plan = pf_plan(pp.SR, pp.SX, pp.ra, pp.rec_slot);
  SALR_CHECK_ARG(plan.total <= kSmemMax, SALR_ERR_CONFIG, "prefill smem plan does not fit");
  pp.w_off = plan.w_off;
  pp.x_off = plan.x_off;
  pp.b_off = plan.b_off;
  pp.rec_off = plan.rec_off;
  pp.bar_off = plan.bar_off;
  const int dev = cur_device();
  static bool attr_done[kMaxDevices] = {};
  if (!attr_done[dev]) {
    SALR_CUDA_TRY(cudaFuncSetAttribute(salr_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    attr_done[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min<int64_t>(sm_count(), pp.items));
  cfg.blockDim = dim3(kPfThreads);
  cfg.dynamicSmemBytes = plan.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  SALR_CUDA_TRY(cudaLaunchKernelEx(&cfg, salr_prefill_kernel, maps[0], maps[1], maps[2], maps[3], pp));
  const int info[12] = {(int)cfg.gridDim.x, pp.SX, 128, -1, pp.ra ? 2 : 0, 0, 0, pdl ? 1 : 0, 0, -1, (int)plan.total, 1};
  for (int i = 0; i < 12; ++i) g_last_launch[i] = info[i];
  return SALR_OK;
}

static inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Workspace layout.  The first kTicketBytes hold the self-resetting ticket
// counters at FIXED offsets (tile tickets, then U tickets) so that calls with
// different shapes sharing one workspace never see stale scratch data there;
// the scratch regions (U hi/lo, U k-split partials, split-K partial tiles)
// follow.
constexpr size_t kTicketBytes = 256 * 1024;
constexpr int64_t kMaxTileTickets = 16 * 1024, kMaxUTickets = 16 * 1024;
constexpr size_t kCtrlOff = kTicketBytes - 64;                 // adapter control words
constexpr size_t kUAccOff = kTicketBytes;                      // 2 parity buffers, fixed place
constexpr size_t kUAccBytes = 2 * (size_t)kUAccElems * 8;
struct WsLayout {
  size_t u_hi, u_lo, u_part, u_tickets, partials, tickets, total;
  int64_t mblocks, ksplit, kchunk, n_tile_tickets;
};
static WsLayout ws_layout(int64_t M, int64_t N, int64_t K, int64_t r_pad, int64_t ctas) {
  WsLayout w = {};
  const int bm = pick_bm(M);
  const int64_t n_mc = (M + bm - 1) / bm, n_nt = (N + kTileN - 1) / kTileN;
  w.n_tile_tickets = n_mc * n_nt;
  w.mblocks = (M + 7) / 8;
  int64_t ks = (2 * (int64_t)sm_count() + w.mblocks - 1) / w.mblocks;
  const int64_t kmax = (K + 31) / 32;
  ks = ks < 1 ? 1 : (ks > kmax ? kmax : ks);
  w.kchunk = (K + ks - 1) / ks;
  w.ksplit = (K + w.kchunk - 1) / w.kchunk;
  w.tickets = 0;
  w.u_tickets = kTicketBytes / 2;
  size_t off = kUAccOff + kUAccBytes;
  w.u_hi = off;
  off += align256((size_t)M * r_pad * 2);
  w.u_lo = off;
  off += align256((size_t)M * r_pad * 2);
  w.u_part = off;
  off += r_pad ? align256((size_t)w.ksplit * M * r_pad * 4) : 0;
  w.partials = off;
  off += align256((size_t)2 * ctas * bm * kTileN * 4);
  w.total = off;
  return w;
}

}  // namespace salr

using namespace salr;

extern "C" {

// Timing instrumentation (tools/trace_linear.py): subsequent launches write
// per-CTA globaltimer stamps into buf[G][32] (u64).  NULL disables.
int salr_debug_set_trace(void* buf) {
  g_trace = static_cast<unsigned long long*>(buf);
  return SALR_OK;
}

int salr_debug_set_probe(void* log, size_t log_words, int max_delay_ns, uint32_t seed) {
  SALR_CHECK_ARG(!log || log_words >= 8, SALR_ERR_CONFIG, "probe log needs >= 8 words");
  SALR_CHECK_ARG(max_delay_ns >= 0 && max_delay_ns <= 1000000, SALR_ERR_CONFIG, "probe delay out of range");
  g_probe_log = static_cast<uint32_t*>(log);
  g_probe_cap = log ? (uint32_t)(log_words - 4) : 0u;
  g_probe_ns = (uint32_t)max_delay_ns;
  g_probe_seed = seed;
  return SALR_OK;
}

int salr_debug_last_launch(int32_t* info12) {
  if (!info12) return SALR_ERR_CONFIG;
  for (int i = 0; i < 12; ++i) info12[i] = g_last_launch[i];
  return SALR_OK;
}

size_t salr_linear_workspace_zero_bytes(void) { return kUAccOff + kUAccBytes; }

// ---- chain workspace: [sync counters][per-linear control + tickets + U] (zero
// once) then the per-linear split-K partial tiles
static constexpr size_t kChainSyncBytes = 4096;
static constexpr size_t kChainCtrlBytes = 256, kChainTicketBytes = 64 * 1024;
static constexpr size_t kChainLinBytes = kChainCtrlBytes + kChainTicketBytes + kUAccBytes;
static constexpr size_t kChainZeroBytes = kChainSyncBytes + kMaxChain * kChainLinBytes;

size_t salr_chain_workspace_zero_bytes(void) { return kChainZeroBytes; }

size_t salr_chain_workspace_bytes(int64_t M, int L) {
  const int bm = pick_bm(M < 1 ? 1 : M);
  return kChainZeroBytes + (size_t)(L < 1 ? 1 : L) * align256((size_t)2 * sm_count() * bm * kTileN * 4);
}

int salr_chain_forward(const salr_chain_linear_t* lin, int L, const void* x0, int64_t M, int64_t ldx0,
                       void* workspace, size_t workspace_bytes, int flags, void* stream) {
  SALR_CHECK_ARG(lin != nullptr && L >= 1 && L <= kMaxChain, SALR_ERR_CONFIG, "chain length %d not in [1, %d]", L,
                 kMaxChain);
  SALR_CHECK_ARG(M >= 1 && M <= 256, SALR_ERR_SHAPE, "chain M=%lld not in [1, 256]", (long long)M);
  SALR_CHECK_ARG(x0 && (reinterpret_cast<uintptr_t>(x0) & 15) == 0 && ldx0 % 8 == 0, SALR_ERR_SHAPE,
                 "x0 must be 16-byte aligned with ldx0 a multiple of 8");
  SALR_CHECK_ARG(workspace_bytes >= salr_chain_workspace_bytes(M, L), SALR_ERR_CONFIG, "workspace too small");
  const int bm = pick_bm(M);
  const int G = sm_count();
  ChainParams cp = {};
  ChainMaps maps;
  memset(&maps, 0, sizeof(maps));
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  cp.L = L;
  cp.M = (int)M;
  cp.n_mc = (int)((M + bm - 1) / bm);
  cp.sync = reinterpret_cast<uint32_t*>(ws);
  int ra_max = 0;
  int64_t rec_max = 0;
  const void* xl = x0;
  int64_t ldxl = ldx0;
  size_t poff = kChainZeroBytes;
  for (int l = 0; l < L; ++l) {
    const salr_chain_linear_t& d = lin[l];
    SALR_CHECK_ARG(d.K >= 1 && d.N >= 1 && d.ldy >= d.N && d.ldy % 8 == 0 && d.y, SALR_ERR_SHAPE,
                   "linear %d: invalid K=%lld N=%lld ldy=%lld", l, (long long)d.K, (long long)d.N, (long long)d.ldy);
    SALR_CHECK_ARG(d.K % 8 == 0 && ldxl >= d.K, SALR_ERR_SHAPE, "linear %d: K=%lld must be a multiple of 8 and <= "
                   "its input's width", l, (long long)d.K);
    SALR_CHECK_ARG(d.r_pad == 0 || ((d.r_pad == 64 || d.r_pad == 128) && d.acat && d.bcat_t), SALR_ERR_CONFIG,
                   "linear %d: r_pad must be 0, 64 or 128 with both factors", l);
    ChainLin& c = cp.l[l];
    c.records = d.records;
    c.tile_off = d.tile_off;
    c.y = d.y;
    c.x = static_cast<const __nv_bfloat16*>(xl);
    c.ldx = (int)ldxl;
    c.acat = static_cast<const __nv_bfloat16*>(d.acat);
    c.N = (int)d.N;
    c.ldy = (int)d.ldy;
    c.K = (int)d.K;
    c.n_kt = (int)((d.K + kTileK - 1) / kTileK);
    c.n_nt = (int)((d.N + kTileN - 1) / kTileN);
    SALR_CHECK_ARG((int64_t)cp.n_mc * c.n_nt <= (int64_t)(kChainTicketBytes / 4) &&
                       (int64_t)cp.n_mc * c.n_nt * c.n_kt < ((int64_t)1 << 31) &&
                       M * (d.ldy > d.N ? d.ldy : d.N) < ((int64_t)1 << 31),
                   SALR_ERR_SHAPE, "linear %d too large for the chain", l);
    c.units = cp.n_mc * c.n_nt * c.n_kt;
    c.ra = (int)(d.r_pad / 64);
    uint8_t* blk = ws + kChainSyncBytes + (size_t)l * kChainLinBytes;
    c.ctrl = reinterpret_cast<uint32_t*>(blk);
    c.tickets = reinterpret_cast<uint32_t*>(blk + kChainCtrlBytes);
    c.u_acc = reinterpret_cast<unsigned long long*>(blk + kChainCtrlBytes + kChainTicketBytes);
    c.partials = reinterpret_cast<float*>(ws + poff);
    poff += align256((size_t)2 * G * bm * kTileN * 4);
    ra_max = std::max(ra_max, c.ra);
    rec_max = std::max<int64_t>(rec_max, d.max_record_bytes > 0 ? d.max_record_bytes : kMaxRecordBytesT2);
    int rc = make_map(&maps.x[l], xl, M, d.K, ldxl, bm);
    if (rc) return rc;
    if (c.ra) {
      const int64_t n_pad = (int64_t)c.n_nt * kTileN;
      if ((rc = make_map(&maps.b[l], d.bcat_t, n_pad, d.r_pad, d.r_pad, kTileN))) return rc;
    } else {
      maps.b[l] = maps.x[l];
    }
    xl = d.y;
    ldxl = d.ldy;
  }
  // every CTA must own units of every linear (the split-K owner arithmetic
  // assumes no empty CTA inside a tile's range): grid <= the smallest linear
  int Gc = G;
  for (int l = 0; l < L; ++l) Gc = std::min(Gc, cp.l[l].units);
  cp.rec_slot = (uint32_t)((std::min<int64_t>(rec_max, kMaxRecordBytesT2) + 16 + 15) & ~15ll);
  cp.stages = 8;
  while (cp.stages > 4 && smem_plan(bm, cp.stages, ra_max, cp.rec_slot).total > kSmemMaxLinear) cp.stages -= 4;
  const SmemPlan plan = smem_plan(bm, cp.stages, ra_max, cp.rec_slot);
  SALR_CHECK_ARG(plan.total <= kSmemMaxLinear, SALR_ERR_CONFIG, "chain ring does not fit shared memory");
  cp.x_off = plan.x_off;
  cp.rec_off = plan.rec_off;
  cp.ad_off = plan.ad_off;
  cp.bar_off = plan.bar_off;
  cp.trace = g_trace;
  const bool pdl = (flags & SALR_FLAG_PDL) != 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto launch = [&](auto kern) -> int {
    const int dev = cur_device();
    static bool attr_done[kMaxDevices][4] = {};
    const int slot = bm == 16 ? 0 : bm == 32 ? 1 : bm == 64 ? 2 : 3;
    if (!attr_done[dev][slot]) {
      SALR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxLinear));
      attr_done[dev][slot] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)Gc);
    cfg.blockDim = dim3(num_threads(4));
    cfg.dynamicSmemBytes = plan.total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    // every CTA waits on the others (Y counters, U slices): co-scheduled, or
    // (programmatic launch, see SALR_FLAG_PDL) checked against occupancy
    if (pdl) {
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, num_threads(4), plan.total) != cudaSuccess) {
        (void)cudaGetLastError();
        per_sm = 1;
      }
      SALR_CHECK_ARG(per_sm >= 1, SALR_ERR_CUDA, "chain grid cannot be co-resident");
    } else {
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SALR_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps, cp));
    return SALR_OK;
  };
  switch (bm) {
    case 16: return launch(salr_chain_kernel<16>);
    case 32: return launch(salr_chain_kernel<32>);
    case 64: return launch(salr_chain_kernel<64>);
    default: return launch(salr_chain_kernel<128>);
  }
}

size_t salr_linear_workspace_bytes(int64_t M, int64_t N, int64_t K, int64_t r_pad, int num_ctas) {
  return ws_layout(M, N, K, r_pad, num_ctas > 0 ? num_ctas : sm_count()).total;
}

int salr_linear_forward(const void* x, int64_t M, int64_t K, int64_t ldx, const uint8_t* records,
                        const uint32_t* tile_off, int64_t max_record_bytes, int64_t N, const void* acat, const void* bcat_t, int64_t r_pad,
                        void* y, int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes, int stages,
                        int num_ctas, int flags, void* stream) {
  SALR_CHECK_ARG(M >= 1 && K >= 1 && N >= 1, SALR_ERR_SHAPE, "invalid dims M=%lld K=%lld N=%lld", (long long)M,
                 (long long)K, (long long)N);
  SALR_CHECK_ARG(ldx >= K && ldx % 8 == 0, SALR_ERR_SHAPE, "ldx=%lld must be >= K and a multiple of 8",
                 (long long)ldx);
  SALR_CHECK_ARG((reinterpret_cast<uintptr_t>(x) & 15) == 0, SALR_ERR_SHAPE, "x must be 16-byte aligned");
  SALR_CHECK_ARG(r_pad == 0 || r_pad == 64 || r_pad == 128, SALR_ERR_CONFIG, "r_pad must be 0, 64 or 128");
  SALR_CHECK_ARG(r_pad == 0 || (acat && bcat_t), SALR_ERR_CONFIG, "adapters need acat and bcat_t");
  const bool nm24 = (flags & SALR_FLAG_NM24) != 0;
  SALR_CHECK_ARG(records && (nm24 || tile_off), SALR_ERR_CONFIG, "records / tile_off missing");
  SALR_CHECK_ARG(y_dtype == kF32 || y_dtype == kBF16, SALR_ERR_DOMAIN, "y dtype must be f32 or bf16");
  SALR_CHECK_ARG(ldy >= N, SALR_ERR_SHAPE, "ldy < N");
  SALR_CHECK_ARG(workspace_bytes >= salr_linear_workspace_bytes(M, N, K, r_pad, num_ctas), SALR_ERR_CONFIG,
                 "workspace too small (%zu < %zu)", workspace_bytes,
                 salr_linear_workspace_bytes(M, N, K, r_pad, num_ctas));
  const int bm = pick_bm(M);
  const int ra = (int)(r_pad / 64);
  const WsLayout wl = ws_layout(M, N, K, r_pad, num_ctas > 0 ? num_ctas : sm_count());
  SALR_CHECK_ARG(wl.n_tile_tickets <= kMaxTileTickets && wl.mblocks * 2 <= kMaxUTickets, SALR_ERR_CONFIG,
                 "problem too large for the ticket area (%lld tiles, %lld m-blocks)", (long long)wl.n_tile_tickets,
                 (long long)wl.mblocks);
  SALR_CHECK_ARG(M * (ldy > N ? ldy : N) < ((int64_t)1 << 31) && M * r_pad < ((int64_t)1 << 31), SALR_ERR_SHAPE,
                 "M x N = %lld x %lld exceeds the 32-bit output index", (long long)M, (long long)N);

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LinearParams p = {};
  p.records = records;
  p.tile_off = tile_off;
  p.y = y;
  p.M = (int)M;
  p.N = (int)N;
  p.ldy = (int)ldy;
  p.n_kt = (int)((K + kTileK - 1) / kTileK);
  p.n_nt = (int)((N + kTileN - 1) / kTileN);
  p.n_mc = (int)((M + bm - 1) / bm);
  SALR_CHECK_ARG((int64_t)p.n_mc * p.n_nt * p.n_kt < ((int64_t)1 << 31), SALR_ERR_SHAPE, "too many work units");
  p.units = p.n_mc * p.n_nt * p.n_kt;
  p.ra = ra;
  p.y_dtype = y_dtype;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = dbg_env("SALR_DEBUG_MODE");
      dbg = e ? atoi(e) : 0;
    }
    p.dbg = dbg;
    p.trace = g_trace;
    p.probe_log = g_probe_log;
    p.probe_cap = g_probe_cap;
    p.probe_ns = g_probe_ns;
    p.probe_seed = g_probe_seed;
  }
  {
    // (the decoders' fixed-width band loads may read a few halfwords past a
    // tile's last value -- into the next slot or the barrier area, never
    // used: the selectors pick zero bytes for absent rows)
    p.rec_slot = nm24 ? (uint32_t)kNmRecBytes
                 : (max_record_bytes > 0 && max_record_bytes <= kMaxRecordBytesT2)
                     ? (uint32_t)((max_record_bytes + 15) & ~15ll) : (uint32_t)kMaxRecordBytesT2;
    p.nm24 = nm24 ? 1 : 0;
    const int smax = max_stages(bm, ra, p.rec_slot, stages > 8 ? std::min(stages, 16) : 8);
    p.stages = stages <= 0 || stages > smax ? smax : stages;
  }
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  p.partials = reinterpret_cast<float*>(ws + wl.partials);
  p.tickets = reinterpret_cast<uint32_t*>(ws + wl.tickets);
  __nv_bfloat16* u_hi = reinterpret_cast<__nv_bfloat16*>(ws + wl.u_hi);
  __nv_bfloat16* u_lo = reinterpret_cast<__nv_bfloat16*>(ws + wl.u_lo);

  CUtensorMap maps[4];
  int rc = make_map(&maps[0], x, M, K, ldx, bm);
  if (rc) return rc;
  if (ra) {
    const int64_t n_pad = (int64_t)p.n_nt * kTileN;
    if ((rc = make_map(&maps[1], bcat_t, n_pad, r_pad, r_pad, kTileN))) return rc;
    if ((rc = make_map(&maps[2], u_hi, M, r_pad, r_pad, bm))) return rc;
    if ((rc = make_map(&maps[3], u_lo, M, r_pad, r_pad, bm))) return rc;
  } else {
    maps[1] = maps[2] = maps[3] = maps[0];
  }

  // Default grid: one persistent CTA per SM, but at least kMinUnitsPerCta
  // units each -- small linears (k/v: 512 units) otherwise pay a deep split-K
  // fixup for a pipeline that never fills.
  constexpr int64_t kMinUnitsPerCta = 6;
  int64_t ctas = num_ctas > 0 ? num_ctas : std::min<int64_t>(sm_count(), (p.units + kMinUnitsPerCta - 1) / kMinUnitsPerCta);
#ifndef SALR_ALIGNED_GRID_MAX_UNITS_SMALL_M
#define SALR_ALIGNED_GRID_MAX_UNITS_SMALL_M 32
#endif
#ifndef SALR_ALIGNED_GRID_MIN_M
#define SALR_ALIGNED_GRID_MIN_M 1
#endif
  if (num_ctas <= 0 && M >= SALR_ALIGNED_GRID_MIN_M && !(dbg_env("SALR_NO_ALIGNED_GRID"))) {
    // Prefer a grid (>= 6/7 of the SMs) whose per-CTA unit ranges tile the
    // K dimension exactly: every split output tile is then shared by
    // CTAs that finish together, so the split-K reduction does not wait on
    // a straggler (q/o/k/v/down at M >= 16, where the reduction is heavy).
    // Also accepted: a grid that is a multiple of the output-tile count --
    // every tile then split over exactly c / tiles CTAs, whose contiguous
    // unit ranges never straddle a tile boundary (q|k|v at M=32: 144 CTAs
    // for 48 tiles, 2.3 us faster than 148).
    const int64_t tiles = p.units / p.n_kt;
    for (int64_t c = ctas; c >= (6 * ctas + 6) / 7; --c) {
      const int64_t per = p.units / c;
      const bool even = p.units % c == 0 && (p.n_kt % per == 0 || per % p.n_kt == 0);
      // below 16 tokens the split-K fixup is cheap: trade SMs for alignment
      // only for short per-CTA ranges (q|k|v, o: ~16-21 units; down's 56
      // units are 2 us slower on 128 CTAs than on 148 at M=1)
      if (M < 16 && per > SALR_ALIGNED_GRID_MAX_UNITS_SMALL_M) break;
      if (even || c % tiles == 0) {
        ctas = c;
        break;
      }
    }
  }
  if (ctas > p.units) ctas = p.units;
  SALR_CHECK_ARG(ctas <= 65535, SALR_ERR_CONFIG, "num_ctas too large");
  // in-kernel U needs every CTA resident at once (they wait on each other's
  // partials): one CTA per SM, grid <= SM count
  // U = X A_cat in-kernel accumulates in int64 fixed point (2^-26, |U| < 2^37);
  // SALR_FLAG_U_FP32 (inputs outside that range) selects the fp32 pre-kernel
  p.u_mode = ra ? ((M <= 256 && ctas <= sm_count() && !(flags & SALR_FLAG_U_FP32)) ? 1 : 2) : 0;
  // cooperative split-tile reduction pays off once a partial tile has rows
  // to share (M >= 16); tiny ones stay with the last CTA (one round trip)
  static const bool no_coop = dbg_env("SALR_NO_COOP") != nullptr;
  p.coop = (ctas <= sm_count() && M >= 16 && !no_coop) ? 1 : 0;
  {
    // Split tiles shared by exactly np (2..8) consecutive CTAs: make those a
    // thread-block cluster and reduce through DSMEM (no global round trips).
    // The partial tile (BM x 128 fp32) reuses the drained ring.  Only when
    // the cooperative reduction is off: with it, the same grid measured
    // ~0.8 us faster per launch (o / down at M=32; the cluster barrier waits
    // for the slowest CTA of the cluster before anyone reduces).
    const int64_t per = p.units / ctas;
    const int64_t np = (p.units % ctas == 0 && per < p.n_kt && p.n_kt % per == 0) ? p.n_kt / per : 0;
    const bool fits = (int64_t)p.stages * (bm * 128 + p.rec_slot) >= (int64_t)(bm + 4) * kTileN * 4;
    static const bool no_cluster = dbg_env("SALR_NO_CLUSTER") != nullptr;
    p.cluster = (!no_cluster && !p.coop && np >= 2 && np <= 8 && ctas % np == 0 && fits) ? (int)np : 0;
  }
  p.K = (int)K;
  p.x = static_cast<const __nv_bfloat16*>(x);
  p.acat = static_cast<const __nv_bfloat16*>(acat);
  p.ldx = (int)ldx;
  p.u_acc = reinterpret_cast<unsigned long long*>(ws + kUAccOff);
  p.ctrl = reinterpret_cast<uint32_t*>(ws + kCtrlOff);
  bool pdl = (flags & SALR_FLAG_PDL) != 0;
  if (p.u_mode == 2) {
    adapter_u_kernel<<<dim3((unsigned)wl.mblocks, (unsigned)wl.ksplit, (unsigned)ra), dim3(64, 4), 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), M, K, ldx, static_cast<const __nv_bfloat16*>(acat), (int)r_pad,
        wl.kchunk, reinterpret_cast<float*>(ws + wl.u_part), reinterpret_cast<uint32_t*>(ws + wl.u_tickets), u_hi,
        u_lo);
    SALR_LAUNCH_CHECK();
    pdl = true;
  }
  static const bool no_prefill = dbg_env("SALR_NO_PREFILL") != nullptr;
  const int64_t pf_items = ((M + 128 * kPfMG - 1) / (128 * kPfMG)) * p.n_nt;
  // The prefill kernel has no split-K: it needs enough (512-token x
  // 128-column) items to occupy the GPU (measured crossover ~3/4 of the SMs).
  // (NM24 matrices always take the decode-size kernel: it covers any M in
  // m-chunks; the prefill kernel reads TB2 only)
  if (M > kPrefillMinM && num_ctas <= 0 && !no_prefill && !nm24 && 4 * pf_items >= 3 * (int64_t)sm_count()) {
    // prefill-size M: decode each weight tile once per 512 tokens
    PrefillParams pp = {};
    pp.records = records;
    pp.tile_off = tile_off;
    pp.y = y;
    pp.y_dtype = y_dtype;
    pp.ldy = (int)ldy;
    pp.M = (int)M;
    pp.N = (int)N;
    pp.n_kt = p.n_kt;
    pp.n_nt = p.n_nt;
    pp.n_mg = (int)((M + 128 * kPfMG - 1) / (128 * kPfMG));
    pp.items = pp.n_mg * pp.n_nt;
    pp.ra = ra;
    pp.rec_slot = p.rec_slot;
    pp.trace = g_trace;
    pp.dbg = p.dbg;
    return launch_prefill(maps, pp, s, pdl);
  }
  if (p.probe_log) {
    SALR_CHECK_ARG(bm == 16, SALR_ERR_CONFIG, "the pipeline probe runs decode-size launches of M <= 16 (M=%lld)",
                   (long long)M);
    return launch_linear_probed(maps, p, (int)ctas, s, pdl);
  }
  switch (bm) {
    case 16: rc = launch_linear<16>(maps, p, (int)ctas, s, pdl); break;
    case 32: rc = launch_linear<32>(maps, p, (int)ctas, s, pdl); break;
    case 64: rc = launch_linear<64>(maps, p, (int)ctas, s, pdl); break;
    default: rc = launch_linear<128>(maps, p, (int)ctas, s, pdl); break;
  }
  return rc;
}

}  // extern "C"
