// Chained SALR linears in one persistent launch (a decode step's layer:
// q|k|v -> o -> gate|up -> down), included by salr_linear.cu.
//
// One launch of salr_linear_kernel per linear pays, every time, the CTA
// start (TMEM allocation, barrier setup, tile-offset and first-record
// latency: ~4 us) and a tail in which SMs sit idle behind the split-K
// reduction (~4-10 us) -- more than half of a 32-layer decode step at M=32.
// Here every CTA walks its stream-K unit range of linear 0, then of linear
// 1, ... with the pipeline running through: the record producer streams the
// next linear's weights as ring slots drain, the decoders expand them, and
// only the X tiles (the previous linear's output) wait -- for a grid-wide
// "Y(l-1) complete" counter that each CTA bumps after its last store of
// Y(l-1).  The roles are those of salr_linear_kernel (warp 0 records, 1 MMA,
// 3 X tiles, 4-19 decoders, 20-23 epilogue); split tiles are reduced by the
// last CTA to publish its partial (no CTA waits on a partner), in CTA order
// as in the single-linear kernel, so results are identical to running the
// linears one by one with the same grid.  In-kernel U = X @ A_cat per linear
// (the same fixed-point slices) once its X is complete.
//
// Dependencies only point from linear l to l+1 and every CTA is resident at
// once (cooperative launch or checked occupancy), so no wait can deadlock:
// the MMA warp reaches linear l+1's units only after all of its linear-l
// units, and the epilogue finishes linear l (stores, reductions, counter)
// before it touches linear l+1 (adapter operands, U).

constexpr int kMaxChain = 4;

struct ChainLin {
  const uint8_t* records;
  const uint32_t* tile_off;
  void* y;                     // bf16, ld ldy
  const __nv_bfloat16* x;      // this linear's input (ld ldx): x0 or the previous y
  const __nv_bfloat16* acat;   // K x 64*ra
  float* partials;             // [2 * G][BM][128] fp32 split-K partial tiles
  uint32_t* tickets;           // n_mc * n_nt, zero on entry and exit
  unsigned long long* u_acc;   // [2][M][64*ra] int64 fixed point (parity-buffered)
  uint32_t* ctrl;              // U control words (as salr_linear_kernel)
  int N, ldy, K, ldx, n_kt, n_nt, units, ra;
};

struct ChainParams {
  ChainLin l[kMaxChain];
  int L, M, n_mc, stages;
  uint32_t rec_slot;
  uint32_t* sync;  // [l]: CTAs done storing Y(l); [kMaxChain]: CTAs finished (zero on entry and exit)
  uint32_t x_off, rec_off, ad_off, bar_off;
  unsigned long long* trace;
};

struct ChainMaps {
  CUtensorMap x[kMaxChain];  // input of linear l (box 64 cols x BM rows)
  CUtensorMap b[kMaxChain];  // B_cat^T of linear l (box 64 x 128)
};

// per-CTA globaltimer stamps (tools/trace_chain.py): slot 8*l + k
#define SALR_CHAIN_TRACE(l, k) \
  do { \
    if (cp.trace) cp.trace[(size_t)blockIdx.x * 32 + 8 * (l) + (k)] = globaltimer(); \
  } while (0)

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int BM>
__global__ void __launch_bounds__(num_threads(4), 1)
    salr_chain_kernel(const __grid_constant__ ChainMaps maps, const ChainParams cp) {
  constexpr int NG = 4;
  constexpr int NACC = nacc_for(BM);
  constexpr int ACOLS = acc_cols_for(BM);
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BM);
  constexpr int kFirstEpi = first_epi_warp(NG);
  constexpr uint32_t a_col0 = (uint32_t)((NACC * ACOLS + 31) & ~31);

  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  const int S = cp.stages;
  uint8_t* xbuf = smem + cp.x_off;
  uint8_t* recbuf = smem + cp.rec_off;
  uint8_t* adbuf = smem + cp.ad_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + cp.bar_off);
  uint64_t* empty = full + S;
  uint64_t* decoded = empty + S;
  uint64_t* xfull = decoded + S;
  uint64_t* acc_full = xfull + S;      // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint64_t* ad_full = acc_empty + 2;
  uint64_t* ad_empty = ad_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ad_empty + 1);
  volatile uint32_t* bcast = tmem_slot + 1;  // epilogue warps' broadcast word

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int bid = blockIdx.x;
  if (threadIdx.x == 0) pdl_launch_dependents();
  auto ub_of = [&](int l) { return (int)((int64_t)bid * cp.l[l].units / G); };
  auto ue_of = [&](int l) { return (int)(((int64_t)bid + 1) * cp.l[l].units / G); };

  if (warp == 0 && lane == 0) {
    for (int l = 0; l < cp.L; ++l) {
      prefetch_tmap(&maps.x[l]);
      if (cp.l[l].ra) prefetch_tmap(&maps.b[l]);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&xfull[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&decoded[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    mbar_init(ad_full, 1);
    mbar_init(ad_empty, 1);
    fence_barrier_init();
  }
  __shared__ __align__(128) uint64_t s_lut[16];
  if (warp == 2 && lane < 16) s_lut[lane] = nib_lut_entry(lane);
  const uint32_t lut_s = smem_u32(s_lut);
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tmem != 0u) __trap();

  if (warp == 0) {
    // ================= record producer: every unit of every linear, in
    // order; weights never wait on data
    int ps = 0, issued = 0;
    uint32_t pph = 0;
    const uint64_t pol = l2_policy_evict_first();
    for (int l = 0; l < cp.L; ++l) {
      const ChainLin& L = cp.l[l];
      const int ub = ub_of(l), ue = ue_of(l), tpm = L.n_nt * L.n_kt;
      for (int c0 = ub; c0 < ue; c0 += 32) {
        // record offsets of 32 units, one coalesced load per lane
        const int v = c0 + (int)lane;
        uint32_t o0 = 0, o1 = 0;
        if (v < ue) {
          const int t = v % tpm;
          o0 = __ldg(L.tile_off + t);
          o1 = __ldg(L.tile_off + t + 1);
        }
        const int n = min(32, ue - c0);
        for (int i = 0; i < n; ++i) {
          const uint32_t a = __shfl_sync(0xffffffffu, o0, i), b = __shfl_sync(0xffffffffu, o1, i);
          if (issued >= S) mbar_wait(&empty[ps], pph ^ 1);
          if (lane == 0) {
            const uint32_t bytes = (b - a) * 16u;
            if (bytes)
              bulk_g2s_hint(recbuf + (size_t)ps * cp.rec_slot, L.records + (size_t)a * 16u, bytes, &full[ps], pol);
            mbar_arrive_expect_tx(&full[ps], bytes);
          }
          __syncwarp();
          if (++ps == S) { ps = 0; pph ^= 1; }
          ++issued;
        }
      }
    }
  } else if (warp == 3) {
    // ================= X producer: linear 0's input may be the preceding
    // kernel's output (programmatic launch); linear l > 0 reads Y(l-1),
    // complete once every CTA has bumped its counter
    pdl_wait();
    int xs = 0, issued = 0;
    uint32_t xph = 0;
    for (int l = 0; l < cp.L; ++l) {
      const ChainLin& L = cp.l[l];
      if (l > 0) {
        if (lane == 0) {
          while (ld_acquire_u32(cp.sync + (l - 1)) < (uint32_t)G) __nanosleep(64);
          fence_proxy_async_global();  // generic-proxy Y stores -> TMA reads
        }
        __syncwarp();
      }
      if (lane == 0) SALR_CHAIN_TRACE(l, 0);
      const int ub = ub_of(l), ue = ue_of(l), tpm = L.n_nt * L.n_kt;
      int kt = ub % L.n_kt, mc = ub / tpm, rem = tpm - ub % tpm;
      for (int v = ub; v < ue; ++v) {
        if (issued >= S) mbar_wait(&empty[xs], xph ^ 1);
        if (lane == 0) {
          tma_2d_g2s(xbuf + (size_t)xs * BM * 128, &maps.x[l], kt * kTileK, mc * BM, &xfull[xs]);
          mbar_arrive_expect_tx(&xfull[xs], BM * 128);
        }
        __syncwarp();
        if (++xs == S) { xs = 0; xph ^= 1; }
        ++issued;
        if (++kt == L.n_kt) kt = 0;
        if (--rem == 0) {
          rem = tpm;
          ++mc;
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one elected lane of the converged warp)
    const uint64_t bdesc0 = desc_kmajor_sw128(smem_u32(xbuf));
    const uint32_t lo0 = (uint32_t)bdesc0, bhi = (uint32_t)(bdesc0 >> 32);
    constexpr uint32_t kLoStep = (uint32_t)(BM * 128) >> 4;
    const uint32_t dec0 = smem_u32(decoded), emp0 = smem_u32(empty), xf0 = smem_u32(xfull);
    int s = 0, seg = 0;
    uint32_t ph = 0, ad_ph = 0;
    for (int l = 0; l < cp.L; ++l) {
      const ChainLin& L = cp.l[l];
      const int ub = ub_of(l), ue = ue_of(l);
      int u = ub;
      while (u < ue) {
        const int tile_base = u - u % L.n_kt;
        const int seg_end = min(ue, tile_base + L.n_kt);
        const int b = NACC == 2 ? (seg & 1) : 0;
        const uint32_t acc_ph = (uint32_t)((NACC == 2 ? seg >> 1 : seg) & 1);
        const uint32_t acc = (uint32_t)(b * ACOLS);
        mbar_wait(&acc_empty[b], acc_ph ^ 1);
        tc_fence_after();
        for (int v = u; v < seg_end; ++v) {
          mbar_wait2_addr(dec0 + 8u * (uint32_t)s, xf0 + 8u * (uint32_t)s, ph);
          tc_fence_after();
          mma_ktile_ts(acc, a_col0 + 32u * (uint32_t)s, lo0 + (uint32_t)s * kLoStep, bhi, IDESC, v != u ? 1u : 0u,
                       emp0 + 8u * (uint32_t)s);
          if (lane == 0 && v == ub) SALR_CHAIN_TRACE(l, 1);
          if (lane == 0 && v == ue - 1) SALR_CHAIN_TRACE(l, 2);
          if (++s == S) { s = 0; ph ^= 1u; }
        }
        if (u == tile_base && L.ra) {
          mbar_wait(ad_full, ad_ph);
          ad_ph ^= 1;
          tc_fence_after();
          if (elect_one()) {
            for (int a = 0; a < L.ra; ++a) {
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
        if (elect_one()) tc_commit(&acc_full[b]);
        __syncwarp();
        ++seg;
        u = seg_end;
      }
    }
  } else if (warp >= kFirstDecWarp && warp < kFirstEpi) {
    // ================= decoders: the concatenated unit sequence of all
    // linears (a decoder needs no per-linear state)
    const int grp = (warp - kFirstDecWarp) >> 2;
    const int q = warp & 3;
    const uint32_t lane_tm = (uint32_t)(32 * q) << 16;
    int total = 0;
    for (int l = 0; l < cp.L; ++l) total += ue_of(l) - ub_of(l);
    int s = grp;
    uint32_t ph = 0;
    for (int it = grp; it < total; it += NG) {
      mbar_wait(&full[s], ph);
      decode_tile_tb2(smem_u32(recbuf + (size_t)s * cp.rec_slot), tmem + lane_tm + a_col0 + 32u * s, q, lane, lut_s);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&decoded[s]);
      s += NG;
      if (s >= S) { s -= S; ph ^= 1; }
    }
  } else if (warp >= kFirstEpi && warp < kFirstEpi + 4) {
    // ================= epilogue (+ in-kernel U, adapter operands, split-K)
    const int q = warp & 3;
    const uint32_t lane_tm = (uint32_t)(32 * q) << 16;
    const int etid = (warp - kFirstEpi) * 32 + (int)lane;
    int seg = 0;
    uint32_t ad_ph = 0;
    bool ad_used = false;  // the adapter slot holds operands an MMA may still read
    constexpr int kSX = kUSlice + 8;
    for (int l = 0; l < cp.L; ++l) {
      const ChainLin& L = cp.l[l];
      const int ub = ub_of(l), ue = ue_of(l), tpm = L.n_nt * L.n_kt;
      const int rp = 64 * L.ra;
      uint32_t par = 0;
      if (L.ra) {
        // ---- U = X @ A_cat (X = x0 or Y(l-1), complete before any slice)
        if (l == 0) {
          pdl_wait();
        } else {
          if (etid == 0) {
            while (ld_acquire_u32(cp.sync + (l - 1)) < (uint32_t)G) __nanosleep(64);
          }
          named_bar_sync(1, 128);
        }
        // the adapter slot doubles as the U staging area: wait until the last
        // adapter MMA of the previous linear has read it
        if (ad_used) {
          if (etid == 0) mbar_wait(ad_empty, ad_ph ^ 1);
          named_bar_sync(1, 128);
        }
        par = *reinterpret_cast<volatile uint32_t*>(L.ctrl + kCtrlEpoch) & 1u;
        unsigned long long* uacc = L.u_acc + (size_t)par * kUAccElems;
        if (bid == 0) {
          unsigned long long* other = L.u_acc + (size_t)(par ^ 1u) * kUAccElems;
          const uint32_t used = L.ctrl[kCtrlUsed + (par ^ 1u)];
          for (uint32_t i = (uint32_t)etid; i < used; i += 128) other[i] = 0ull;
          if (etid == 0) {
            L.ctrl[kCtrlReady + (par ^ 1u)] = 0u;
            L.ctrl[kCtrlSlice + (par ^ 1u)] = 0u;
            L.ctrl[kCtrlUsed + (par ^ 1u)] = 0u;
            L.ctrl[kCtrlUsed + par] = (uint32_t)(cp.M * rp);
          }
        }
        const int kSA = rp + 8;
        const int nsl = (L.K + kUSlice - 1) / kUSlice;
        __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(adbuf);
        __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(adbuf + (uint32_t)kUSlice * kSA * 2u);
        const uint32_t sa_u = smem_u32(sa), sx_u = smem_u32(sx);
        int sl = bid;
        while (sl < nsl) {
          const int k0 = sl * kUSlice, ks = min(kUSlice, L.K - k0), ks16 = (ks + 15) & ~15;
          {
            const int cpr = rp / 8;
            const __nv_bfloat16* src = L.acat + (size_t)k0 * rp;
            for (int i = etid; i < ks16 * cpr; i += 128) {
              const int kr = i / cpr, c = i % cpr;
              cp_async_16(smem_u32(sa + kr * kSA + 8 * c), src + (size_t)(kr < ks ? i : 0) * 8, kr < ks ? 16u : 0u);
            }
          }
          const int wid = etid >> 5;
          const int g = (int)lane >> 2, t = (int)lane & 3;
          for (int m0 = 0; m0 < cp.M; m0 += BM) {
            const int rows = min(BM, cp.M - m0);
            if (m0) named_bar_sync(1, 128);
            for (int i = etid; i < rows * (ks16 / 8); i += 128) {
              const int m = i / (ks16 / 8), c = i % (ks16 / 8);
              cp_async_16(smem_u32(sx + m * kSX + 8 * c), L.x + (size_t)(m0 + m) * L.ldx + k0 + (c < ks / 8 ? 8 * c : 0),
                          c < ks / 8 ? 16u : 0u);
            }
            cp_async_wait_all();
            named_bar_sync(1, 128);
            const int nnb = rp / 8, items = nnb * ((rows + 15) / 16);
            for (int itm = wid; itm < items; itm += 4) {
              const int nb = itm % nnb, mb = itm / nnb;
              float c4[4] = {0.f, 0.f, 0.f, 0.f};
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
                mma_m16n8k16_bf16(c4, af, bf);
              }
              const int r0 = mb * 16 + g, n = nb * 8 + 2 * t;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int r = r0 + 8 * h;
                if (r < rows) {
                  unsigned long long* dst = uacc + (size_t)(m0 + r) * rp + n;
                  atomicAdd(dst, (unsigned long long)__float2ll_rn(c4[2 * h] * (float)(1ll << kUFrac)));
                  atomicAdd(dst + 1, (unsigned long long)__float2ll_rn(c4[2 * h + 1] * (float)(1ll << kUFrac)));
                }
              }
            }
          }
          named_bar_sync(1, 128);  // every partial of this slice issued; staging reusable
          if (etid == 0) {
            fence_acq_rel_gpu();
            atomicAdd(L.ctrl + kCtrlReady + par, 1u);
            *bcast = (uint32_t)G + atomicAdd(L.ctrl + kCtrlSlice + par, 1u);
          }
          named_bar_sync(1, 128);
          sl = (int)*bcast;
          named_bar_sync(1, 128);
        }
        if (etid == 0) {
          while (ld_acquire_u32(L.ctrl + kCtrlReady + par) < (uint32_t)nsl) __nanosleep(32);
        }
        named_bar_sync(1, 128);
      }
      // ---- adapter operands of a first-k segment into the adapter slot:
      // B_cat^T tile by TMA, U hi/lo (BM x 64 per rank block, K-major, 128B
      // swizzle) from the fixed-point U
      auto prep_adapter = [&](int useg) {
        const int nt = (useg / L.n_kt) % L.n_nt;
        const int mc = useg / tpm;
        if (etid == 0) {
          mbar_wait(ad_empty, ad_ph ^ 1);
          for (int a = 0; a < L.ra; ++a)
            tma_2d_g2s(adbuf + (size_t)a * (kAdTileBytes + 2u * BM * 128u), &maps.b[l], 64 * a, nt * kTileN, ad_full);
        }
        named_bar_sync(1, 128);
        const unsigned long long* uacc = L.u_acc + (size_t)par * kUAccElems;
        for (int e = etid; e < BM * 32 * L.ra; e += 128) {
          const int a = e / (BM * 32);
          const int m = (e / 32) % BM;
          const int rr = 2 * (e % 32);
          const int gm = mc * BM + m;
          float u0 = 0.f, u1 = 0.f;
          if (gm < cp.M) {
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
        named_bar_sync(1, 128);
        if (etid == 0) mbar_arrive_expect_tx(ad_full, (uint32_t)L.ra * kAdTileBytes);
        ad_ph ^= 1;
        ad_used = true;
      };
      auto next_first_k = [&](int from) {
        const int t = from % L.n_kt == 0 ? from : from - from % L.n_kt + L.n_kt;
        return t < ue ? t : ue;
      };
      int next_ad = L.ra ? next_first_k(ub) : ue;
      if (next_ad < ue) {
        prep_adapter(next_ad);
        next_ad = next_first_k(next_ad + 1);
      }
      // ---- segments: drain the accumulator to Y (whole output tile) or to
      // this CTA's partial slot (split tile)
      int u = ub;
      while (u < ue) {
        const int tile_base = u - u % L.n_kt;
        const int seg_end = min(ue, tile_base + L.n_kt);
        const bool full_cover = (u == tile_base) && (seg_end == tile_base + L.n_kt);
        const int nt = (u / L.n_kt) % L.n_nt;
        const int mc = u / tpm;
        const int b = NACC == 2 ? (seg & 1) : 0;
        const uint32_t acc_ph = (uint32_t)((NACC == 2 ? seg >> 1 : seg) & 1);
        mbar_wait_backoff(&acc_full[b], acc_ph, 256);
        tc_fence_after();
        if (etid == 0 && u == ub) SALR_CHAIN_TRACE(l, 5);
        float* part_tile = L.partials + ((size_t)bid * 2 + (u == ub ? 0 : 1)) * (size_t)BM * kTileN;
        const int nl = 32 * q + (int)lane;
        const int n = nt * kTileN + nl;
        const bool n_ok = n < L.N;
        const int rows = min(BM, cp.M - mc * BM);
        const size_t yrow0 = (size_t)(mc * BM) * L.ldy + n;
#pragma unroll 1
        for (int c0 = 0; c0 < rows; c0 += 8) {
          uint32_t r[8];
          SALR_TMEM_LD_X8(tmem + lane_tm + (uint32_t)(b * ACOLS + c0), r);
          tc_wait_ld();
          if (!full_cover) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c0 + i < rows) __stcg(part_tile + (size_t)(c0 + i) * kTileN + nl, __uint_as_float(r[i]));
          } else if (n_ok) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (c0 + i < rows)
                static_cast<__nv_bfloat16*>(L.y)[yrow0 + (size_t)(c0 + i) * L.ldy] =
                    __float2bfloat16_rn(__uint_as_float(r[i]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[b]);
        if (next_ad < ue && u == tile_base) {
          prep_adapter(next_ad);
          next_ad = next_first_k(next_ad + 1);
        }
        ++seg;
        u = seg_end;
      }
      if (etid == 0) SALR_CHAIN_TRACE(l, 6);
      // ---- split-K tail: publish this CTA's partials (one release, one
      // acq_rel ticket per split tile); the CTA completing a ticket sums the
      // tile's partials in CTA order and writes it -- nobody waits
      int tl[2];
      int nsplit = 0;
      if (ub < ue) {
        const int t0 = ub - ub % L.n_kt, t1 = (ue - 1) - (ue - 1) % L.n_kt;
        if (!(t0 >= ub && t0 + L.n_kt <= ue)) tl[nsplit++] = t0;
        if (t1 != t0 && !(t1 >= ub && t1 + L.n_kt <= ue)) tl[nsplit++] = t1;
      }
      named_bar_sync(1, 128);  // every partial and Y store of this CTA issued (CTA scope)
      if (etid == 0) {
        uint32_t lf = 0;
        for (int j = 0; j < nsplit; ++j) {
          const int tb = tl[j];
          const int np = cta_of(tb + L.n_kt - 1, L.units, G) - cta_of(tb, L.units, G) + 1;
          const uint32_t old = ticket_add_acq_rel(&L.tickets[(tb / tpm) * L.n_nt + (tb / L.n_kt) % L.n_nt], 1u);
          if (old + 1 == (uint32_t)np) lf |= 1u << j;
        }
        *bcast = lf;
        SALR_CHAIN_TRACE(l, 3);
      }
      named_bar_sync(1, 128);
      const uint32_t lf = *bcast;
#ifdef SALR_CHAIN_DEBUG
      if (etid == 0 && (bid < 3 || bid > G - 3))
        printf("cta %d l %d ub %d ue %d nsplit %d lf %u tl0 %d N %d ldy %d y %p\n", bid, l, ub, ue, nsplit, lf,
               nsplit ? tl[0] : -1, L.N, L.ldy, L.y);
#endif
      for (int j = 0; j < nsplit; ++j) {
        if (!((lf >> j) & 1u)) continue;
        const int tb = tl[j];
        const int ntb = (tb / L.n_kt) % L.n_nt, mcb = tb / tpm;
        const int rows = min(BM, cp.M - mcb * BM);
        const int c_first = cta_of(tb, L.units, G), c_last = cta_of(tb + L.n_kt - 1, L.units, G);
        const int cb_first = (int)((int64_t)c_first * L.units / G);
        const size_t tile_elems = (size_t)BM * kTileN;
        const float* p_first = L.partials + ((size_t)c_first * 2 + (cb_first >= tb ? 0 : 1)) * tile_elems;
        // kIPT 4-column chunks per thread and pass, partials of up to 4 CTAs
        // per batch: every load of a batch is in flight before any sum (one
        // L2 round trip per batch), sums in CTA order
        constexpr int kIPT = 4, kCB = 4;
        const int items = rows * (kTileN / 4);
        __nv_bfloat16* yy = static_cast<__nv_bfloat16*>(L.y);
        for (int e0 = etid; e0 < items; e0 += 128 * kIPT) {
          float4 acc[kIPT];
          size_t offs[kIPT];
#pragma unroll
          for (int i = 0; i < kIPT; ++i) {
            const int e = e0 + i * 128;
            const int m = e / (kTileN / 4), c4 = 4 * (e % (kTileN / 4));
            offs[i] = (size_t)m * kTileN + c4;
            if (e < items) acc[i] = __ldcg(reinterpret_cast<const float4*>(p_first + offs[i]));
          }
          for (int c = c_first + 1; c <= c_last; c += kCB) {
            float4 vv[kCB][kIPT];
#pragma unroll
            for (int j = 0; j < kCB; ++j)
#pragma unroll
              for (int i = 0; i < kIPT; ++i)
                if (c + j <= c_last && e0 + i * 128 < items)
                  vv[j][i] = __ldcg(reinterpret_cast<const float4*>(L.partials + (size_t)(c + j) * 2 * tile_elems +
                                                                    offs[i]));
#pragma unroll
            for (int j = 0; j < kCB; ++j)
#pragma unroll
              for (int i = 0; i < kIPT; ++i)
                if (c + j <= c_last && e0 + i * 128 < items) {
                  acc[i].x += vv[j][i].x;
                  acc[i].y += vv[j][i].y;
                  acc[i].z += vv[j][i].z;
                  acc[i].w += vv[j][i].w;
                }
          }
#pragma unroll
          for (int i = 0; i < kIPT; ++i) {
            const int e = e0 + i * 128;
            if (e >= items) continue;
            const int m = e / (kTileN / 4), c4 = 4 * (e % (kTileN / 4));
            const int col = ntb * kTileN + c4;
            const size_t o = (size_t)(mcb * BM + m) * L.ldy + col;
            if (col < L.N) yy[o] = __float2bfloat16_rn(acc[i].x);
            if (col + 1 < L.N) yy[o + 1] = __float2bfloat16_rn(acc[i].y);
            if (col + 2 < L.N) yy[o + 2] = __float2bfloat16_rn(acc[i].z);
            if (col + 3 < L.N) yy[o + 3] = __float2bfloat16_rn(acc[i].w);
          }
        }
        if (etid == 0) L.tickets[mcb * L.n_nt + ntb] = 0u;
      }
      if (etid == 0) SALR_CHAIN_TRACE(l, 4);
      // ---- Y(l) done on this CTA (stores, reductions): release the counter
      // the next linear's X tiles and U wait for; U epoch ticket
      named_bar_sync(1, 128);
      if (etid == 0) {
        fence_proxy_async_global();
        fence_acq_rel_gpu();
        atomicAdd(cp.sync + l, 1u);
        SALR_CHAIN_TRACE(l, 7);
        if (L.ra) {
          const uint32_t d = atomicAdd(L.ctrl + kCtrlDone, 1u);
          if (d + 1 == (uint32_t)G) {
            L.ctrl[kCtrlDone] = 0u;
            fence_acq_rel_gpu();
            L.ctrl[kCtrlEpoch] = L.ctrl[kCtrlEpoch] + 1u;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (threadIdx.x == 0) {
    // the last CTA out resets the Y-done counters for the next launch (every
    // CTA has passed all its waits on them)
    fence_acq_rel_gpu();
    if (atomicAdd(cp.sync + kMaxChain, 1u) + 1 == (uint32_t)G) {
      for (int l = 0; l < cp.L; ++l) cp.sync[l] = 0u;
      cp.sync[kMaxChain] = 0u;
      fence_acq_rel_gpu();
    }
  }
}
