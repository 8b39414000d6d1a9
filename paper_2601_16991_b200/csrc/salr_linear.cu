// SALR linear forward on sm_100a:  Y = X @ decode(W) + (X @ A_cat) @ B_cat
//
// Reference: pkg/src/salr/pipeline.py:405-461 (pipelined_forward: stage-1
// bitmap decode into tiles, stage-2 tile products, adapter delta added once),
// pkg/src/salr/fusion.py:87-92 (apply_fused: exactly two products).
//
// B200 design:
//   * swap-AB: the tensor core computes Y^T tile = W^T tile (128 output cols,
//     M_mma = 128) x X^T (N_mma = BM tokens) with the fp32 accumulator in TMEM.
//   * stage 1 (decode) is a producer warpgroup: decoder thread (warp q, lane
//     l) owns output column n = 32q + l of the tile == TMEM lane 32q + l and
//     expands that column's bitmap bits into bf16 pairs along K, written
//     straight into TMEM with tcgen05.st -- the A operand of tcgen05.mma is
//     read from TMEM, so decoded tiles never touch shared memory.
//   * TMA: one warp streams each compressed tile record (1-D bulk copy) and
//     the matching X tile (2-D tensor map, 128B swizzle) into a ring of
//     STAGES shared-memory slots (full/empty mbarriers, expect_tx).
//   * one thread issues tcgen05.mma; tcgen05.commit frees the ring slot and
//     the TMEM A stage, so decode of tile k+1 overlaps the MMA of tile k (the
//     GPU form of the reference's SPSC ring, pipeline.py:110-183).
//   * adapters: U = X @ A_cat is produced by a small pre-kernel (PDL
//     overlapped); the CTA that owns k-tile 0 of an output tile adds
//     B_cat^T x U^T (hi + lo bf16 split of U) into the SAME TMEM accumulator,
//     so Y leaves the chip once.
//   * stream-K: every CTA owns a contiguous range of (m-chunk, n-tile, k-tile)
//     work units; a CTA that covers only part of an output tile's K range
//     stores its fp32 partial tile, and the last CTA to finish that tile sums
//     the partials in a fixed CTA order -- results are bit-identical from run
//     to run (the reference's schedule-independence, pipeline.py:1-13).
#include <cstdint>
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
  const __nv_bfloat16* bcat_t;  // (n_nt*128) x r_pad, or nullptr
  const float* u;               // M x r_pad fp32 (X @ A_cat), or nullptr
  void* y;
  float* partials;              // [2 * gridDim.x][BM][128] fp32 split-K partial tiles
  uint32_t* tickets;            // n_mc * n_nt, zero on entry and exit
  int M, N, ldy;                // 32-bit indexing: host checks M * max(N, ldy) < 2^31
  int n_kt, n_nt, n_mc;
  int units;                    // n_mc * n_nt * n_kt
  int r_pad;                    // 0, 64 or 128
  int y_dtype;
  int stages;                   // ring slots in use, 1 (serial) .. stages_for(BM)
};

constexpr int kRecSlot = kMaxRecordBytesBf16;  // 17424, multiple of 16
constexpr int kTmemCols = 512;
constexpr int kAccCol = 0;
constexpr int kAStageCol = 256;                // A stage s at 256 + 32 s

__host__ __device__ constexpr int stages_for(int bm) { return bm <= 64 ? 6 : (bm <= 128 ? 4 : 3); }

struct SmemPlan {
  uint32_t x_off, u_off, rec_off, bar_off, total;
};
__host__ __device__ inline SmemPlan smem_plan(int bm, int stages, int r_pad) {
  SmemPlan p;
  p.x_off = 0;
  p.u_off = p.x_off + stages * bm * 128;
  const int ra = r_pad / 64;
  p.rec_off = p.u_off + 2 * ra * bm * 128;
  p.bar_off = p.rec_off + stages * kRecSlot;
  p.bar_off = (p.bar_off + 15) & ~15u;
  p.total = p.bar_off + 8 * (3 * stages + 3) + 16 + 1024;  // + slack for 1024 alignment
  return p;
}

// CTA that owns work unit u under the even contiguous split of `units` over `ctas`.
__device__ __forceinline__ int cta_of(int u, int units, int ctas) {
  return (int)((((int64_t)u + 1) * ctas + units - 1) / units - 1);
}

template <int BM, int NDEC>
__global__ void __launch_bounds__(128 + NDEC * 32, 1)
    salr_linear_kernel(const __grid_constant__ CUtensorMap xmap, const LinearParams p) {
  constexpr int STAGES = stages_for(BM);
  constexpr int NPART = NDEC / 4;            // decoder warps per TMEM lane quarter
  constexpr int RP = kTileK / NPART;         // rows (K) per decoder warp
  constexpr int ACOLS = RP / 2;              // TMEM columns written per decoder warp
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BM);
  static_assert(NDEC % 4 == 0 && (ACOLS == 8 || ACOLS == 16 || ACOLS == 32), "decoder split");

  extern __shared__ uint8_t smem_raw[];
  // 128B-swizzled TMA/UMMA tiles need 1024-byte alignment; pad by an offset
  // (not a pointer round-trip) so the compiler keeps the shared address space
  // and emits 32-bit LDS.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const SmemPlan plan = smem_plan(BM, STAGES, p.r_pad);
  uint8_t* xbuf = smem + plan.x_off;
  uint8_t* ubuf = smem + plan.u_off;
  uint8_t* recbuf = smem + plan.rec_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + plan.bar_off);
  uint64_t* empty = full + STAGES;
  uint64_t* decoded = empty + STAGES;
  uint64_t* acc_full = decoded + STAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* ad_ready = acc_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ad_ready + 1);
  volatile uint32_t* last_flag = tmem_slot + 1;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;

  // ---- per-CTA work range
  const int G = gridDim.x;
  const int u_begin = (int)((int64_t)blockIdx.x * p.units / G);
  const int u_end = (int)(((int64_t)blockIdx.x + 1) * p.units / G);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&xmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&decoded[s], NDEC);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, NDEC);
    mbar_init(ad_ready, NDEC);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= TMA producer
    if (lane == 0) {
      int it = 0;
      for (int u = u_begin; u < u_end; ++u, ++it) {
        const int s = (int)(it % p.stages);
        const uint32_t ph = (uint32_t)((it / p.stages) & 1);
        mbar_wait(&empty[s], ph ^ 1);
        const int kt = u % p.n_kt;
        const int nt = (u / p.n_kt) % p.n_nt;
        const int mc = u / (p.n_kt * p.n_nt);
        const int t = nt * p.n_kt + kt;
        const uint32_t o0 = p.tile_off[t], o1 = p.tile_off[t + 1];
        const uint32_t bytes = (o1 - o0) * 16u;
        mbar_arrive_expect_tx(&full[s], bytes + BM * 128);
        bulk_g2s(recbuf + (size_t)s * kRecSlot, p.records + (size_t)o0 * 16u, bytes, &full[s]);
        tma_2d_g2s(xbuf + (size_t)s * BM * 128, &xmap, (int32_t)(kt * kTileK), (int32_t)(mc * BM), &full[s]);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread)
    if (lane == 0) {
      int it = 0, seg = 0;
      uint32_t ad_phase = 0;
      int u = u_begin;
      while (u < u_end) {
        const int tile_base = u - u % p.n_kt;
        const int seg_end = min(u_end, tile_base + p.n_kt);
        const bool first_k = (u == tile_base);
        mbar_wait(acc_empty, (uint32_t)(seg & 1) ^ 1u);
        tc_fence_after();
        for (int v = u; v < seg_end; ++v, ++it) {
          const int s = (int)(it % p.stages);
          const uint32_t ph = (uint32_t)((it / p.stages) & 1);
          mbar_wait(&full[s], ph);
          mbar_wait(&decoded[s], ph);
          tc_fence_after();
          const uint64_t bdesc = desc_kmajor_sw128(smem_u32(xbuf + (size_t)s * BM * 128));
          const uint32_t a_tm = tmem + kAStageCol + 32 * s;
#pragma unroll
          for (int j = 0; j < kTileK / 16; ++j)
            mma_ts(tmem + kAccCol, a_tm + 8 * j, bdesc + 2 * j, IDESC, (v != u || j) ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        if (first_k && p.r_pad > 0) {
          mbar_wait(ad_ready, ad_phase);
          ad_phase ^= 1u;
          tc_fence_after();
          const int ra = p.r_pad / 64;
          const uint32_t ad_tm = tmem + kAStageCol + 32 * STAGES;
          for (int half = 0; half < 2; ++half) {
            for (int a = 0; a < ra; ++a) {
              const uint64_t ud = desc_kmajor_sw128(smem_u32(ubuf + (size_t)(half * ra + a) * BM * 128));
#pragma unroll
              for (int j = 0; j < 4; ++j) mma_ts(tmem + kAccCol, ad_tm + 32 * a + 8 * j, ud + 2 * j, IDESC, 1u);
            }
          }
        }
        tc_commit(acc_full);
        ++seg;
        u = seg_end;
      }
    }
  } else if (warp >= 4) {
    // ================= decoders (+ adapter staging + epilogue)
    const int dw = warp - 4;
    const int q = warp & 3;            // TMEM lane quarter == 32-column group
    const int part = dw >> 2;          // which RP-row slice of the tile
    const uint32_t lt = lanemask_lt();
    const uint32_t lanebit = 1u << lane;
    const uint32_t lane_tm = (uint32_t)(32 * q) << 16;
    int it = 0, seg = 0;
    bool pdl_done = false;
    int u = u_begin;
    while (u < u_end) {
      const int tile_base = u - u % p.n_kt;
      const int seg_end = min(u_end, tile_base + p.n_kt);
      const bool first_k = (u == tile_base);
      const bool full_cover = first_k && (seg_end == tile_base + p.n_kt);
      const int nt = (u / p.n_kt) % p.n_nt;
      const int mc = u / (p.n_kt * p.n_nt);

      for (int v = u; v < seg_end; ++v, ++it) {
        const int s = (int)(it % p.stages);
        const uint32_t ph = (uint32_t)((it / p.stages) & 1);
        mbar_wait(&full[s], ph);
        const uint8_t* rec = recbuf + s * kRecSlot;
        const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec);
        const uint32_t* gbits = hdr + 4 + q * kTileK;         // this group's 64 row words
        const uint16_t* vals = reinterpret_cast<const uint16_t*>(rec + kValOffset);
        // this warp's RP row words (broadcast loads, all issued up front)
        uint32_t w[RP];
#pragma unroll
        for (int i = 0; i < RP; i += 4) {
          const uint4 q4 = *reinterpret_cast<const uint4*>(gbits + part * RP + i);
          w[i] = q4.x; w[i + 1] = q4.y; w[i + 2] = q4.z; w[i + 3] = q4.w;
        }
        uint32_t off = q == 0 ? 0u : hdr[q - 1];
        if (part > 0) {  // values of this group in the rows before this slice
          uint32_t c = 0u;
          for (int k = (int)lane; k < part * RP; k += 32) c += __popc(gbits[k]);
          off += __reduce_add_sync(0xffffffffu, c);
        }
        uint32_t packed[ACOLS];
        const uint16_t* vp = vals + off;  // first value of the current row
#pragma unroll
        for (int k2 = 0; k2 < ACOLS; ++k2) {
          const uint32_t w0 = w[2 * k2], w1 = w[2 * k2 + 1];
          const uint16_t* vp1 = vp + __popc(w0);
          uint32_t v0 = 0u, v1 = 0u;
          if (w0 & lanebit) v0 = vp[__popc(w0 & lt)];
          if (w1 & lanebit) v1 = vp1[__popc(w1 & lt)];
          vp = vp1 + __popc(w1);
          packed[k2] = __byte_perm(v0, v1, 0x5410);
        }
        const uint32_t taddr = tmem + lane_tm + kAStageCol + 32 * s + ACOLS * part;
        tmem_st_cols<ACOLS>(taddr, packed);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&decoded[s]);
      }

      if (first_k && p.r_pad > 0) {
        if (!pdl_done) {
          pdl_wait();  // U = X @ A_cat comes from the preceding kernel
          pdl_done = true;
        }
        const int ra = p.r_pad / 64;
        // B_cat^T rows -> TMEM adapter A operand (this warp: lane quarter q, column slice `part`)
        {
          const int n = nt * kTileN + 32 * q + lane;
          const uint32_t* src = reinterpret_cast<const uint32_t*>(p.bcat_t + (size_t)n * p.r_pad);
          const int cols = p.r_pad / 2;                  // u32 columns of this row
          const int per = cols / NPART;
          const uint32_t ad_tm = tmem + lane_tm + kAStageCol + 32 * STAGES + per * part;
          for (int c = 0; c < per; c += 8) {
            uint32_t r[8];
#pragma unroll
            for (int i = 0; i < 8; i += 4) {
              const uint4 q4 = __ldg(reinterpret_cast<const uint4*>(src + per * part + c + i));
              r[i] = q4.x; r[i + 1] = q4.y; r[i + 2] = q4.z; r[i + 3] = q4.w;
            }
            tmem_st_cols<8>(ad_tm + c, r);
          }
        }
        // U (fp32) -> bf16 hi/lo, K-major 128B-swizzled B operand tiles in smem
        {
          const int pairs = BM * (p.r_pad / 2);
          for (int i = dw * 32 + (int)lane; i < pairs; i += NDEC * 32) {
            const int m = i / (p.r_pad / 2);
            const int r = 2 * (i % (p.r_pad / 2));
            const int gm = mc * BM + m;
            float2 uv = make_float2(0.f, 0.f);
            if (gm < p.M) uv = *reinterpret_cast<const float2*>(p.u + (size_t)gm * p.r_pad + r);
            const __nv_bfloat16 h0 = __float2bfloat16_rn(uv.x), h1 = __float2bfloat16_rn(uv.y);
            const __nv_bfloat16 l0 = __float2bfloat16_rn(uv.x - __bfloat162float(h0));
            const __nv_bfloat16 l1 = __float2bfloat16_rn(uv.y - __bfloat162float(h1));
            const int a = r / 64, rr = r % 64;
            const int chunk = (rr * 2) / 16, within = (rr * 2) % 16;
            const uint32_t boff = (uint32_t)(m * 128 + ((chunk ^ (m & 7)) * 16) + within);
            __nv_bfloat162 hv = __halves2bfloat162(h0, h1), lv = __halves2bfloat162(l0, l1);
            *reinterpret_cast<__nv_bfloat162*>(ubuf + (size_t)a * BM * 128 + boff) = hv;
            *reinterpret_cast<__nv_bfloat162*>(ubuf + (size_t)(ra + a) * BM * 128 + boff) = lv;
          }
        }
        fence_proxy_async_smem();
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ad_ready);
      }

      // ---- epilogue: accumulator columns [part*BM/NPART, (part+1)*BM/NPART)
      mbar_wait(acc_full, (uint32_t)(seg & 1));
      tc_fence_after();
      // partial slot of this CTA: 0 for its first segment, 1 otherwise
      float* part_tile = p.partials + ((size_t)blockIdx.x * 2 + (u == u_begin ? 0 : 1)) * (size_t)BM * kTileN;
      {
        constexpr int CPW = BM / NPART;   // columns (tokens) per warp
        const int nl = 32 * q + (int)lane;
        const int n = nt * kTileN + nl;
        const bool n_ok = n < p.N;
        for (int c0 = 0; c0 < CPW; c0 += 16) {
          uint32_t r[16];
          const int col = part * CPW + c0;
          SALR_TMEM_LD_X16(tmem + lane_tm + kAccCol + col, r);
          tc_wait_ld();
          const int lim = CPW < 16 ? CPW : 16;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i >= lim) break;
            const float val = __uint_as_float(r[i]);
            if (full_cover) {
              const int m = mc * BM + col + i;
              if (!n_ok || m >= p.M) continue;
              if (p.y_dtype == kF32) static_cast<float*>(p.y)[(size_t)m * p.ldy + n] = val;
              else static_cast<__nv_bfloat16*>(p.y)[(size_t)m * p.ldy + n] = __float2bfloat16_rn(val);
            } else {
              __stcg(part_tile + (size_t)(col + i) * kTileN + nl, val);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);

      if (!full_cover) {
        // stream-K fixup: the last CTA to finish this (m-chunk, n-tile) sums
        // the partial tiles of CTAs c_first..c_last in that fixed order.
        __threadfence();
        named_bar_sync(1, NDEC * 32);
        const int a = tile_base;
        const int c_first = cta_of(a, p.units, G), c_last = cta_of(a + p.n_kt - 1, p.units, G);
        if (dw == 0 && lane == 0) {
          const uint32_t old = atomicAdd(&p.tickets[mc * p.n_nt + nt], 1u);
          *last_flag = (old + 1 == (uint32_t)(c_last - c_first + 1)) ? 1u : 0u;
        }
        named_bar_sync(1, NDEC * 32);
        if (*last_flag) {
          __threadfence();
          const int tid = dw * 32 + (int)lane;
          const int nl = tid % kTileN;
          const int n = nt * kTileN + nl;
          for (int mm = tid / kTileN; mm < BM; mm += NDEC * 32 / kTileN) {
            const int m = mc * BM + mm;
            if (m >= p.M || n >= p.N) continue;
            float acc = 0.0f;
            for (int c = c_first; c <= c_last; ++c) {
              const int cb = (int)((int64_t)c * p.units / G);  // u_begin of CTA c
              const float* pt = p.partials + ((size_t)c * 2 + (cb >= a ? 0 : 1)) * (size_t)BM * kTileN;
              acc += __ldcg(pt + (size_t)mm * kTileN + nl);
            }
            if (p.y_dtype == kF32) static_cast<float*>(p.y)[(size_t)m * p.ldy + n] = acc;
            else static_cast<__nv_bfloat16*>(p.y)[(size_t)m * p.ldy + n] = __float2bfloat16_rn(acc);
          }
          if (tid == 0) p.tickets[mc * p.n_nt + nt] = 0u;
        }
        named_bar_sync(1, NDEC * 32);
      }
      ++seg;
      u = seg_end;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// U[m, r] = sum_k X[m, k] * A_cat[k, r] (fp32).  Grid (m-blocks of 8 rows,
// K splits, r blocks of 64); every block stores its partial, and the last
// block of each (m-block, r-block) -- found with a self-resetting ticket --
// sums the K-split partials in split order, so U is bit-reproducible.
__global__ void __launch_bounds__(256) adapter_u_kernel(const __nv_bfloat16* __restrict__ x, int64_t M, int64_t K,
                                                        int64_t ldx, const __nv_bfloat16* __restrict__ acat,
                                                        int r_pad, int64_t kchunk, float* __restrict__ u_part,
                                                        uint32_t* __restrict__ u_tickets, float* __restrict__ u) {
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
  __threadfence();
  __syncthreads();
  uint32_t* ticket = u_tickets + (size_t)blockIdx.x * gridDim.z + blockIdx.z;
  if (threadIdx.x == 0 && ty == 0) is_last = (atomicAdd(ticket, 1u) + 1 == gridDim.y) ? 1u : 0u;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int j = 0; j < 2; ++j) {
    const int64_t m = j ? mb : ma;
    if (m >= M) continue;
    float sum = 0.f;
    for (unsigned ks = 0; ks < gridDim.y; ++ks) sum += __ldcg(u_part + (size_t)ks * M * r_pad + m * r_pad + r);
    u[m * r_pad + r] = sum;
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

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BM>
static int launch_linear(const CUtensorMap& xmap, const LinearParams& p, int ctas, cudaStream_t s, bool pdl) {
  constexpr int NDEC = 16;
  auto kern = salr_linear_kernel<BM, NDEC>;
  const SmemPlan plan = smem_plan(BM, stages_for(BM), p.r_pad);
  SALR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.total));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(128 + NDEC * 32);
  cfg.dynamicSmemBytes = plan.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  SALR_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, xmap, p));
  return SALR_OK;
}

static inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

static int pick_bm(int64_t M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return 256;
}

// Workspace layout.  The first kTicketBytes hold the self-resetting ticket
// counters at FIXED offsets (tile tickets, then U tickets) so that calls with
// different shapes sharing one workspace never see stale scratch data there;
// the scratch regions (U, U k-split partials, split-K partial tiles) follow.
constexpr size_t kTicketBytes = 256 * 1024;
constexpr int64_t kMaxTileTickets = 32 * 1024, kMaxUTickets = 32 * 1024;
struct WsLayout {
  size_t u, u_part, u_tickets, partials, tickets, total;
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
  size_t off = kTicketBytes;
  w.u = off;
  off += align256((size_t)M * r_pad * 4);
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

size_t salr_linear_workspace_bytes(int64_t M, int64_t N, int64_t K, int64_t r_pad, int num_ctas) {
  return ws_layout(M, N, K, r_pad, num_ctas > 0 ? num_ctas : sm_count()).total;
}

int salr_linear_forward(const void* x, int64_t M, int64_t K, int64_t ldx, const uint8_t* records,
                        const uint32_t* tile_off, int64_t N, const void* acat, const void* bcat_t, int64_t r_pad,
                        void* y, int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes, int stages,
                        int num_ctas, void* stream) {
  SALR_CHECK_ARG(M >= 1 && K >= 1 && N >= 1, SALR_ERR_SHAPE, "invalid dims M=%lld K=%lld N=%lld", (long long)M,
                 (long long)K, (long long)N);
  SALR_CHECK_ARG(ldx >= K && ldx % 8 == 0, SALR_ERR_SHAPE, "ldx=%lld must be >= K and a multiple of 8",
                 (long long)ldx);
  SALR_CHECK_ARG((reinterpret_cast<uintptr_t>(x) & 15) == 0, SALR_ERR_SHAPE, "x must be 16-byte aligned");
  SALR_CHECK_ARG(r_pad == 0 || r_pad == 64 || r_pad == 128, SALR_ERR_CONFIG, "r_pad must be 0, 64 or 128");
  SALR_CHECK_ARG(r_pad == 0 || (acat && bcat_t), SALR_ERR_CONFIG, "adapters need acat and bcat_t");
  SALR_CHECK_ARG(y_dtype == kF32 || y_dtype == kBF16, SALR_ERR_DOMAIN, "y dtype must be f32 or bf16");
  SALR_CHECK_ARG(ldy >= N, SALR_ERR_SHAPE, "ldy < N");
  SALR_CHECK_ARG(workspace_bytes >= salr_linear_workspace_bytes(M, N, K, r_pad, num_ctas), SALR_ERR_CONFIG,
                 "workspace too small (%zu < %zu)", workspace_bytes,
                 salr_linear_workspace_bytes(M, N, K, r_pad, num_ctas));
  const int bm = pick_bm(M);
  SALR_CHECK_ARG(!(bm == 256 && r_pad > 64), SALR_ERR_CONFIG, "r_pad=128 needs M <= 128 per chunk");
  {
    const WsLayout w0 = ws_layout(M, N, K, r_pad, num_ctas > 0 ? num_ctas : sm_count());
    SALR_CHECK_ARG(w0.n_tile_tickets <= kMaxTileTickets && w0.mblocks * 2 <= kMaxUTickets, SALR_ERR_CONFIG,
                   "problem too large for the ticket area (%lld tiles, %lld m-blocks)",
                   (long long)w0.n_tile_tickets, (long long)w0.mblocks);
  }
  EncodeTiledFn enc = get_encode_tiled();
  SALR_CHECK_ARG(enc != nullptr, SALR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  LinearParams p = {};
  p.records = records;
  p.tile_off = tile_off;
  p.bcat_t = static_cast<const __nv_bfloat16*>(bcat_t);
  p.y = y;
  SALR_CHECK_ARG(M * (ldy > N ? ldy : N) < ((int64_t)1 << 31) && M * r_pad < ((int64_t)1 << 31), SALR_ERR_SHAPE,
                 "M x N = %lld x %lld exceeds the 32-bit output index", (long long)M, (long long)N);
  p.M = (int)M;
  p.N = (int)N;
  p.ldy = (int)ldy;
  p.n_kt = (int)((K + kTileK - 1) / kTileK);
  p.n_nt = (int)((N + kTileN - 1) / kTileN);
  p.n_mc = (int)((M + bm - 1) / bm);
  SALR_CHECK_ARG((int64_t)p.n_mc * p.n_nt * p.n_kt < ((int64_t)1 << 31), SALR_ERR_SHAPE, "too many work units");
  p.units = p.n_mc * p.n_nt * p.n_kt;
  p.r_pad = (int)r_pad;
  p.y_dtype = y_dtype;
  {
    const int smax = stages_for(bm);
    p.stages = stages <= 0 || stages > smax ? smax : stages;
  }
  const WsLayout wl = ws_layout(M, N, K, r_pad, num_ctas > 0 ? num_ctas : sm_count());
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  float* u = reinterpret_cast<float*>(ws + wl.u);
  p.partials = reinterpret_cast<float*>(ws + wl.partials);
  p.tickets = reinterpret_cast<uint32_t*>(ws + wl.tickets);
  p.u = r_pad ? u : nullptr;

  CUtensorMap xmap;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kTileK, (cuuint32_t)bm};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SALR_CHECK_ARG(cr == CUDA_SUCCESS, SALR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);

  bool pdl = false;
  if (r_pad) {
    adapter_u_kernel<<<dim3((unsigned)wl.mblocks, (unsigned)wl.ksplit, (unsigned)(r_pad / 64)), dim3(64, 4), 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), M, K, ldx, static_cast<const __nv_bfloat16*>(acat), (int)r_pad,
        wl.kchunk, reinterpret_cast<float*>(ws + wl.u_part), reinterpret_cast<uint32_t*>(ws + wl.u_tickets), u);
    SALR_LAUNCH_CHECK();
    pdl = true;
  }
  int64_t ctas = num_ctas > 0 ? num_ctas : sm_count();
  if (ctas > p.units) ctas = p.units;
  SALR_CHECK_ARG(ctas <= 65535, SALR_ERR_CONFIG, "num_ctas too large");
  int rc;
  switch (bm) {
    case 16: rc = launch_linear<16>(xmap, p, (int)ctas, s, pdl); break;
    case 32: rc = launch_linear<32>(xmap, p, (int)ctas, s, pdl); break;
    case 64: rc = launch_linear<64>(xmap, p, (int)ctas, s, pdl); break;
    case 128: rc = launch_linear<128>(xmap, p, (int)ctas, s, pdl); break;
    default: rc = launch_linear<256>(xmap, p, (int)ctas, s, pdl); break;
  }
  return rc;
}

}  // extern "C"
