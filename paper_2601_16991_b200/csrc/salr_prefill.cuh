// Prefill-size SALR linear (M > 256 tokens): decode each weight tile ONCE per
// 512 tokens.  Included by salr_linear.cu inside namespace salr (shares the
// TB2 format, PTX helpers and host plumbing).
//
// The decode-size kernel (salr_linear_kernel) re-decodes every weight tile
// for every 128-token chunk, so at M = 2048 it decodes the matrix 16 times.
// Here the MMA is not swapped: D[128 tokens x 128 cols] += X[128 x 64] .
// W[64 x 128], both operands K-major in shared memory.  A work item is one
// 128-column output tile for MG = 4 token chunks (512 tokens): per 64-row
// k-step the 16 decoder warps expand the record ONCE into a K-major SW128
// W^T tile in shared memory (a lane = one output column = one 128-byte row,
// exactly the decoder's natural order), and the MMA warp issues 4 x 4
// tcgen05.mma (one per token chunk) into four 128-column TMEM accumulators
// (all 512 columns).  Adapters: two (hi/lo) extra k-steps per r-block with
// U tiles in the X ring and the B_cat^T tile in its own slot.  Tensor time
// per k-step (16 MMAs, ~1k cycles) exceeds the decode time, so the kernel is
// MMA-bound, as prefill should be.
//
// Rings (mbarrier pairs, one phase per use):
//   records  SR slots  producer -> decoders          rec_full / rec_empty
//   W tiles  2 slots   decoders -> MMA               w_full (16 arrivals) / w_empty
//   X tiles  SX slots  producer -> MMA               x_full / x_empty
//   B_cat    1 slot    producer -> MMA (per item)    b_full / b_empty
//   accum    1         MMA -> epilogue (per item)    acc_full / acc_empty (4 arrivals)

constexpr int kPfMG = 4;                   // 128-token chunks per work item
constexpr int kPfThreads = 768;            // 24 warps
constexpr int kPfTile = 128 * 128;         // bytes of one K-major 128x64 bf16 operand tile
constexpr int kPfDecWarp0 = 4, kPfEpiWarp0 = 20;

struct PrefillParams {
  const uint8_t* records;     // TB2 records
  const uint32_t* tile_off;   // TB2 offsets (16-byte units), n_nt * n_kt + 1
  void* y;
  int y_dtype, ldy, M, N, n_kt, n_nt, n_mg, items, ra;
  uint32_t rec_slot;
  int SR, SX;
  uint32_t w_off, x_off, b_off, rec_off, bar_off;
  unsigned long long* trace;  // tools only: CTA 0 per-step globaltimer stamps [4][64]
  int dbg;                    // experiments: 1 skip decode, 8 skip MMAs (wrong results)
};
#define PF_TRACE(ev, i)                                                                    \
  do {                                                                                     \
    if (p.trace && blockIdx.x == 0 && (i) < 64) p.trace[(ev) * 64 + (i)] = globaltimer(); \
  } while (0)

struct PfPlan {
  uint32_t w_off, x_off, b_off, rec_off, bar_off, total;
};
inline PfPlan pf_plan(int SR, int SX, int ra, uint32_t rec_slot) {
  PfPlan p;
  p.w_off = 0;                                   // 2 x W tile (1024-aligned pieces first)
  p.x_off = p.w_off + 2u * kPfTile;              // SX x X/U tile
  p.b_off = p.x_off + (uint32_t)SX * kPfTile;    // ra x B_cat^T tile
  p.rec_off = p.b_off + (uint32_t)ra * kPfTile;  // SR x record slot
  p.bar_off = p.rec_off + (uint32_t)SR * rec_slot;
  p.bar_off = (p.bar_off + 7u) & ~7u;
  p.total = p.bar_off + 8u * (2u * SR + 2u * SX + 8u) + 16u + 1024u;
  return p;
}

__global__ void __launch_bounds__(kPfThreads, 1)
    salr_prefill_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap bmap,
                        const __grid_constant__ CUtensorMap uhimap, const __grid_constant__ CUtensorMap ulomap,
                        const PrefillParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* wbuf = smem + p.w_off;
  uint8_t* xbuf = smem + p.x_off;
  uint8_t* bbuf = smem + p.b_off;
  uint8_t* recbuf = smem + p.rec_off;
  const int SR = p.SR, SX = p.SX;
  uint64_t* rec_full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* rec_empty = rec_full + SR;
  uint64_t* x_full = rec_empty + SR;
  uint64_t* x_empty = x_full + SX;
  uint64_t* w_full = x_empty + SX;  // [2]
  uint64_t* w_empty = w_full + 2;   // [2]
  uint64_t* b_full = w_empty + 2;
  uint64_t* b_empty = b_full + 1;
  uint64_t* acc_full = b_empty + 1;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int G = gridDim.x;
  if (threadIdx.x == 0) pdl_launch_dependents();
  auto item_geom = [&](int it, int& mg, int& nt, int& mgc) {
    mg = it / p.n_nt;
    nt = it % p.n_nt;
    const int rows_left = p.M - mg * kPfMG * 128;
    mgc = min(kPfMG, (rows_left + 127) / 128);
  };

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&xmap);
      if (p.ra) {
        prefetch_tmap(&bmap);
        prefetch_tmap(&uhimap);
        prefetch_tmap(&ulomap);
      }
      for (int s = 0; s < SR; ++s) {
        mbar_init(&rec_full[s], 1);
        mbar_init(&rec_empty[s], 16);
      }
      for (int s = 0; s < SX; ++s) {
        mbar_init(&x_full[s], 1);
        mbar_init(&x_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&w_full[s], 16);
        mbar_init(&w_empty[s], 1);
      }
      mbar_init(b_full, 1);
      mbar_init(b_empty, 1);
      mbar_init(acc_full, 1);
      mbar_init(acc_empty, 4);
      fence_barrier_init();
    }
  } else if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================= producer: records (weights, before the PDL wait is
    // irrelevant here: U and X may come from the preceding kernels)
    pdl_wait();
    const uint64_t pol = l2_policy_evict_first();
    int rs = 0;
    uint32_t rph = 0, bph = 0;
    for (int it = blockIdx.x; it < p.items; it += G) {
      int mg, nt, mgc;
      item_geom(it, mg, nt, mgc);
      if (p.ra) {
        if (lane == 0) {
          mbar_wait(b_empty, bph ^ 1);
          for (int a = 0; a < p.ra; ++a) tma_2d_g2s(bbuf + (size_t)a * kPfTile, &bmap, a * 64, nt * 128, b_full);
          mbar_arrive_expect_tx(b_full, (uint32_t)p.ra * kPfTile);
        }
        bph ^= 1;
      }
      const uint32_t* toff = p.tile_off + (size_t)nt * p.n_kt;
      for (int k0 = 0; k0 < p.n_kt; k0 += 32) {
        // 32 record offsets per coalesced load
        const int kk = k0 + (int)lane;
        const uint32_t o0 = kk < p.n_kt ? __ldg(toff + kk) : 0u;
        const uint32_t o1 = kk < p.n_kt ? __ldg(toff + kk + 1) : 0u;
        for (int k = k0; k < min(p.n_kt, k0 + 32); ++k) {
          const uint32_t a0 = __shfl_sync(0xffffffffu, o0, k - k0);
          const uint32_t a1 = __shfl_sync(0xffffffffu, o1, k - k0);
          if (lane == 0) {
            mbar_wait(&rec_empty[rs], rph ^ 1);
            const uint32_t bytes = (a1 - a0) * 16u;
            if (bytes) bulk_g2s_hint(recbuf + (size_t)rs * p.rec_slot, p.records + (size_t)a0 * 16u, bytes, &rec_full[rs], pol);
            mbar_arrive_expect_tx(&rec_full[rs], bytes);
            PF_TRACE(0, k);
          }
          __syncwarp();
          if (++rs == SR) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp == 2) {
    // ================= X producer (token tiles, then U tiles per item): its
    // own warp so the record ring runs ahead independently of the X ring
    pdl_wait();
    int xs = 0;
    uint32_t xph = 0;
    if (lane == 0) {
      for (int it = blockIdx.x; it < p.items; it += G) {
        int mg, nt, mgc;
        item_geom(it, mg, nt, mgc);
        const int row0 = mg * kPfMG * 128;
        for (int k = 0; k < p.n_kt; ++k)
          for (int c = 0; c < mgc; ++c) {
            mbar_wait(&x_empty[xs], xph ^ 1);
            tma_2d_g2s(xbuf + (size_t)xs * kPfTile, &xmap, k * 64, row0 + c * 128, &x_full[xs]);
            mbar_arrive_expect_tx(&x_full[xs], kPfTile);
            if (++xs == SX) { xs = 0; xph ^= 1; }
          }
        if (p.ra)
          for (int h = 0; h < 2; ++h)
            for (int a = 0; a < p.ra; ++a)
              for (int c = 0; c < mgc; ++c) {
                mbar_wait(&x_empty[xs], xph ^ 1);
                tma_2d_g2s(xbuf + (size_t)xs * kPfTile, h ? &ulomap : &uhimap, a * 64, row0 + c * 128, &x_full[xs]);
                mbar_arrive_expect_tx(&x_full[xs], kPfTile);
                if (++xs == SX) { xs = 0; xph ^= 1; }
              }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================= MMA issuer (one elected lane of the converged warp)
    constexpr uint32_t IDESC = idesc_bf16_f32(128, 128);
    int xs = 0, ws = 0;
    uint32_t xph = 0, wph = 0, bph = 0, aph = 0;
    for (int it = blockIdx.x; it < p.items; it += G) {
      int mg, nt, mgc;
      item_geom(it, mg, nt, mgc);
      mbar_wait(acc_empty, aph ^ 1);
      tc_fence_after();
      for (int k = 0; k < p.n_kt; ++k) {
        mbar_wait(&w_full[ws], wph);
        if (lane == 0) PF_TRACE(3, k);
        tc_fence_after();
        const uint64_t wdesc = desc_kmajor_sw128(smem_u32(wbuf + (size_t)ws * kPfTile));
        for (int c = 0; c < mgc; ++c) {
          mbar_wait(&x_full[xs], xph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t xdesc = desc_kmajor_sw128(smem_u32(xbuf + (size_t)xs * kPfTile));
            if (!(p.dbg & 8)) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                mma_ss(tmem + 128u * c, xdesc + 2 * j, wdesc + 2 * j, IDESC, (k | j) ? 1u : 0u);
            }
            tc_commit(&x_empty[xs]);
          }
          __syncwarp();
          if (++xs == SX) { xs = 0; xph ^= 1; }
        }
        if (elect_one()) {
          tc_commit(&w_empty[ws]);
          PF_TRACE(2, k);
        }
        __syncwarp();
        if (++ws == 2) { ws = 0; wph ^= 1; }
      }
      if (p.ra) {
        mbar_wait(b_full, bph);
        tc_fence_after();
        for (int h = 0; h < 2; ++h)
          for (int a = 0; a < p.ra; ++a) {
            const uint64_t bdesc = desc_kmajor_sw128(smem_u32(bbuf + (size_t)a * kPfTile));
            for (int c = 0; c < mgc; ++c) {
              mbar_wait(&x_full[xs], xph);
              tc_fence_after();
              if (elect_one()) {
                const uint64_t udesc = desc_kmajor_sw128(smem_u32(xbuf + (size_t)xs * kPfTile));
#pragma unroll
                for (int j = 0; j < 4; ++j) mma_ss(tmem + 128u * c, udesc + 2 * j, bdesc + 2 * j, IDESC, 1u);
                tc_commit(&x_empty[xs]);
              }
              __syncwarp();
              if (++xs == SX) { xs = 0; xph ^= 1; }
            }
          }
        if (elect_one()) tc_commit(b_empty);
        __syncwarp();
        bph ^= 1;
      }
      if (elect_one()) tc_commit(acc_full);
      __syncwarp();
      aph ^= 1;
    }
  } else if (warp >= kPfDecWarp0 && warp < kPfEpiWarp0) {
    // ================= decoders: all 16 warps expand one record per k-step.
    // Warp (part, q): output columns 32q..32q+31 (one per lane) and bands
    // 4*part..4*part+3 (k rows 16*part..16*part+15) -> two 16-byte chunks of
    // the lane's 128-byte K-major row of the W^T tile (128B swizzle).
    const int dw = warp - kPfDecWarp0;
    const int q = warp & 3;
    const int part = dw >> 2;
    const int n = 32 * q + (int)lane;  // row of the W^T tile
    int rs = 0, ws = 0;
    uint32_t rph = 0, wph = 0;
    for (int it = blockIdx.x; it < p.items; it += G) {
      for (int k = 0; k < p.n_kt; ++k) {
        mbar_wait(&rec_full[rs], rph);
        mbar_wait(&w_empty[ws], wph ^ 1);
        const uint8_t* rec = recbuf + (size_t)rs * p.rec_slot;
        if (p.dbg & 1) {
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&w_full[ws]);
            mbar_arrive(&rec_empty[rs]);
          }
          if (++rs == SR) { rs = 0; rph ^= 1; }
          if (++ws == 2) { ws = 0; wph ^= 1; }
          continue;
        }
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
        uint32_t packed[8];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {  // compile-time bands for this warp's part
          if (pp != part) continue;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int b = 4 * pp + i;
            const uint32_t ev = e[(b >= 8 ? 2 : 0) + (b & 1)];
            const uint32_t ex = (ev >> (8 * ((b & 7) >> 1))) & 0xFFu;
            const uint32_t bov = (bo[b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
            uint32_t r = vbase + 2u * (bov + ex);
            const uint32_t word = b < 8 ? mw.x : mw.y;
            const int sh = 4 * (b & 7);
            uint32_t v0 = 0u, v1 = 0u, v2 = 0u, v3 = 0u;
            asm volatile(
                "{\n\t.reg .pred q0, q1, q2, q3;\n\t"
                "setp.ne.b32 q0, %5, 0;\n\t"
                "setp.ne.b32 q1, %6, 0;\n\t"
                "setp.ne.b32 q2, %7, 0;\n\t"
                "setp.ne.b32 q3, %8, 0;\n\t"
                "@q0 ld.shared.u16 %0, [%4];\n\t"
                "@q0 add.u32 %4, %4, 2;\n\t"
                "@q1 ld.shared.u16 %1, [%4];\n\t"
                "@q1 add.u32 %4, %4, 2;\n\t"
                "@q2 ld.shared.u16 %2, [%4];\n\t"
                "@q2 add.u32 %4, %4, 2;\n\t"
                "@q3 ld.shared.u16 %3, [%4];\n\t}"
                : "+r"(v0), "+r"(v1), "+r"(v2), "+r"(v3), "+r"(r)
                : "r"(word & (1u << sh)), "r"(word & (2u << sh)), "r"(word & (4u << sh)), "r"(word & (8u << sh)));
            packed[2 * i] = __byte_perm(v0, v1, 0x5410);
            packed[2 * i + 1] = __byte_perm(v2, v3, 0x5410);
          }
        }
        // k rows 16*part .. +15 = 16-byte chunks 2*part, 2*part+1 of row n
        uint8_t* wrow = wbuf + (size_t)ws * kPfTile + (size_t)(n >> 3) * 1024 + (size_t)(n & 7) * 128;
        const int c0 = 2 * part, sw = n & 7;
        *reinterpret_cast<uint4*>(wrow + 16 * (c0 ^ sw)) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        *reinterpret_cast<uint4*>(wrow + 16 * ((c0 + 1) ^ sw)) = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&w_full[ws]);
          mbar_arrive(&rec_empty[rs]);
          if (dw == 0) PF_TRACE(1, k);
        }
        if (++rs == SR) { rs = 0; rph ^= 1; }
        if (++ws == 2) { ws = 0; wph ^= 1; }
      }
    }
  } else if (warp >= kPfEpiWarp0) {
    // ================= epilogue: warp q drains TMEM lanes 32q.. (token rows)
    const int q = warp & 3;
    uint32_t aph = 0;
    for (int it = blockIdx.x; it < p.items; it += G) {
      int mg, nt, mgc;
      item_geom(it, mg, nt, mgc);
      while (!mbar_test_wait(acc_full, aph)) __nanosleep(256);
      tc_fence_after();
      for (int c = 0; c < mgc; ++c) {
        const int row = mg * kPfMG * 128 + c * 128 + 32 * q + (int)lane;
        for (int col0 = 0; col0 < 128; col0 += 16) {
          uint32_t r[16];
          SALR_TMEM_LD_X16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(128 * c + col0), r);
          tc_wait_ld();
          if (row >= p.M) continue;
          const int n0 = nt * 128 + col0;
          const size_t o = (size_t)row * p.ldy + n0;
          if (p.y_dtype == kF32) {
            float* yo = static_cast<float*>(p.y) + o;
            if (n0 + 16 <= p.N && (p.ldy & 3) == 0) {
#pragma unroll
              for (int v = 0; v < 4; ++v)
                reinterpret_cast<uint4*>(yo)[v] = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
            } else {
              for (int i = 0; i < 16 && n0 + i < p.N; ++i) yo[i] = __uint_as_float(r[i]);
            }
          } else {
            __nv_bfloat16* yo = static_cast<__nv_bfloat16*>(p.y) + o;
            if (n0 + 16 <= p.N && (p.ldy & 7) == 0) {
              uint32_t h[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const __nv_bfloat162 t2 = __floats2bfloat162_rn(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
                h[i] = *reinterpret_cast<const uint32_t*>(&t2);
              }
              reinterpret_cast<uint4*>(yo)[0] = make_uint4(h[0], h[1], h[2], h[3]);
              reinterpret_cast<uint4*>(yo)[1] = make_uint4(h[4], h[5], h[6], h[7]);
            } else {
              for (int i = 0; i < 16 && n0 + i < p.N; ++i) yo[i] = __float2bfloat16_rn(__uint_as_float(r[i]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      aph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}
