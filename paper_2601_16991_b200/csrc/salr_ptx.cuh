// Thin inline-PTX helpers for sm_100a: mbarriers, bulk/tensor TMA, tcgen05
// (TMEM alloc/ld/st, MMA, commit), descriptors.  Written for this project;
// no CUTLASS dependency.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>

namespace salr {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Suspend-time hint of the blocking waits (ns): a waiting warp is parked until
// the phase completes or the hint elapses, so long waits cost few re-polls.
#ifndef SALR_WAIT_HINT_NS
#define SALR_WAIT_HINT_NS 100000
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "n"(SALR_WAIT_HINT_NS)
      : "memory");
  return ok != 0;
}
// Non-suspending probe of phase completion.
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// Blocking wait: try_wait lets the hardware park the warp until the phase
// completes (or a time limit), so waiting warps do not burn issue slots that
// the decoder warps need.  Debug builds (-DSALR_DEBUG) bound every wait: a
// protocol bug traps (a launch error the host maps to SalrError) instead of
// hanging the device -- the GPU form of the reference ring's wait timeout
// (pipeline.py:59-60, 131-136).
#ifdef SALR_DEBUG
#ifndef SALR_WAIT_TIMEOUT_NS
#define SALR_WAIT_TIMEOUT_NS 2000000000ull
#endif
__device__ __forceinline__ unsigned long long salr_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void salr_wait_timeout(uint32_t bar, uint32_t phase) {
  printf("salr: mbarrier wait timed out (block %d thread %d, barrier 0x%x, parity %u)\n", (int)blockIdx.x,
         (int)threadIdx.x, bar, phase);
  __trap();
}
#define SALR_BOUNDED_WAIT(cond, bar, phase)                                              \
  do {                                                                                   \
    const unsigned long long t0_ = salr_gtimer();                                        \
    while (!(cond)) {                                                                    \
      if (salr_gtimer() - t0_ > SALR_WAIT_TIMEOUT_NS) salr_wait_timeout((bar), (phase)); \
    }                                                                                    \
  } while (0)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if defined(SALR_WAIT_SPIN)
  while (!mbar_test_wait(bar, phase)) {
  }
#elif defined(SALR_DEBUG)
  SALR_BOUNDED_WAIT(mbar_try_wait(bar, phase), smem_u32(bar), phase);
#else
  while (!mbar_try_wait(bar, phase)) {
  }
#endif
}
// Long, latency-tolerant waits (an epilogue warp idle for a whole output
// tile): poll with a plain nanosleep backoff.  A suspended try_wait is woken
// by every mbarrier update of the CTA (hundreds per microsecond in the decode
// pipeline), so a warp parked in it for ~20 us re-polls hundreds of times
// and takes issue slots from the decoders on its SM sub-partition; the
// backoff bounds that to ~1 poll per max_ns at <= max_ns added latency.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t phase, uint32_t max_ns) {
  uint32_t ns = 32;
  while (!mbar_test_wait(bar, phase)) {
    __nanosleep(ns);
    ns = ns < max_ns ? 2 * ns : max_ns;
  }
}
// Spinning wait (no suspension) for very short expected waits.
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t phase) {
  while (!mbar_test_wait(bar, phase)) {
  }
}

// One lane of a fully active warp (the same lane every call): lets the
// compiler keep warp-uniform operands of tcgen05/TMA instructions in uniform
// registers instead of re-broadcasting them from a divergent lane-0 branch.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Warpgroup register re-balancing (all 4 warps of a warpgroup execute it).
template <uint32_t R>
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R));
}
template <uint32_t R>
__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R));
}

// ---------------------------------------------------------------- proxies / PDL
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 16-bit shared-memory load by 32-bit shared address, zero-extended.
// volatile: stays ordered after the (volatile) mbarrier waits that publish
// the TMA-written data.
__device__ __forceinline__ uint32_t lds_u16(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

// Warp-level bf16 MMA m16n8k16 (fp32 accumulate) for the small adapter
// product U = X A_cat, where a tcgen05 tile would be mostly padding.
__device__ __forceinline__ void mma_m16n8k16_bf16(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// 16-byte global -> shared copy (LDGSTS); src_bytes < 16 zero-fills the rest.
__device__ __forceinline__ void cp_async_16(uint32_t dst_smem, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_smem), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------- TMA
// 1-D bulk copy global -> shared, completion on an mbarrier (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same, with an L2 cache-policy hint (createpolicy): the weight records are
// read exactly once per launch, so they stream through L2 as evict-first and
// leave the small, reused data (tile offsets, X, U, adapters) resident.
__device__ __forceinline__ void bulk_g2s_hint(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 32-bit global load through L2 with a cache policy (read-only data)
__device__ __forceinline__ uint32_t ld_u32_hint(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// 2-D tiled tensor copy global -> shared (box defined by the tensor map).
__device__ __forceinline__ void tma_2d_g2s(void* dst_smem, const CUtensorMap* map, int32_t c0,
                                           int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst_smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// prmt.b32 (default mode): selector nibbles are used as given (the CUDA
// __byte_perm intrinsic masks them with 0x7777 first: one more instruction)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// Shared-memory loads by 32-bit shared address (the decoders keep record
// addresses as shared-window offsets; "memory" keeps them behind the
// mbarrier waits that publish the data).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u16z(uint32_t a) {  // zero-extended
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 lds_v2_u32(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds_v4_u32(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
// Funnel shifts of the 64-bit {hi:lo} right by n (wrap: n mod 32; clamp: min(n, 32)).
__device__ __forceinline__ uint32_t shf_r_wrap(uint32_t lo, uint32_t hi, uint32_t n) {
  uint32_t d;
  asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(hi), "r"(n));
  return d;
}
__device__ __forceinline__ uint32_t shf_r_clamp(uint32_t lo, uint32_t hi, uint32_t n) {
  uint32_t d;
  asm("shf.r.clamp.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(hi), "r"(n));
  return d;
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem-desc]^T, kind::f16 (bf16 in, fp32 accumulate), cta_group::1
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[smem-desc] * B[smem-desc]^T, kind::f16, cta_group::1
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32-bit, N consecutive columns per thread.
#define SALR_TMEM_ST_X16(taddr, r)                                                                    \
  asm volatile(                                                                                       \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16};" ::"r"(taddr),                                                                       \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),         \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])   \
      : "memory")

#define SALR_TMEM_LD_X16(taddr, r)                                                                    \
  asm volatile(                                                                                       \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"   \
      "%15}, [%16];"                                                                                  \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),      \
        "=r"(r[14]), "=r"(r[15])                                                                      \
      : "r"(taddr)                                                                                    \
      : "memory")

#define SALR_TMEM_LD_X8(taddr, r)                                                                    \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"               \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
                 "=r"(r[7])                                                                           \
               : "r"(taddr)                                                                           \
               : "memory")

#define SALR_TMEM_ST_X8(taddr, r)                                                                \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),  \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])  \
               : "memory")

// Store N (multiple of 8) consecutive 32-bit TMEM columns of this thread's lane.
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t* r) {
  if constexpr (N % 16 == 0) {
#pragma unroll
    for (int c = 0; c < N; c += 16) SALR_TMEM_ST_X16(taddr + c, (r + c));
  } else {
#pragma unroll
    for (int c = 0; c < N; c += 8) SALR_TMEM_ST_X8(taddr + c, (r + c));
  }
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row core-matrix
// groups 1024 B apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t desc_kmajor_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                      // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // SBO
  d |= (uint64_t)1 << 46;                      // version
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}

// Address-form mbarrier waits (the caller keeps barrier addresses in
// registers and advances them incrementally).
__device__ __forceinline__ void mbar_wait_addr(uint32_t bar, uint32_t phase) {
#if defined(SALR_WAIT_SPIN)
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
#elif defined(SALR_DEBUG)
  auto try_once = [&]() {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase), "n"(SALR_WAIT_HINT_NS)
        : "memory");
    return ok != 0;
  };
  SALR_BOUNDED_WAIT(try_once(), bar, phase);
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(bar),
      "r"(phase), "n"(SALR_WAIT_HINT_NS)
      : "memory");
#endif
}
// Wait for two barriers at once (same parity): both probes are in flight
// together, so the waiter pays one probe latency, not two.
__device__ __forceinline__ void mbar_wait2_addr(uint32_t bar0, uint32_t bar1, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p0, p1;\n\t"
      "W_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p0, [%0], %2;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p1, [%1], %2;\n\t"
      "and.pred p0, p0, p1;\n\t"
      "@!p0 bra W_%=;\n\t}" ::"r"(bar0),
      "r"(bar1), "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint32_t mbar_test_addr(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok;
}
// One k-tile of the main MMA chain, issued by one elected lane of a
// converged warp: 4 x (M=128, K=16) MMAs with A (the decoded W^T tile) in
// TMEM at a_tm and B (the X tile, K-major SW128) described by {lo, hi},
// then a commit to the stage's empty barrier.  accumulate == 0 starts the
// accumulator.  Everything in one asm block: no per-MMA descriptor
// arithmetic in C, no divergent region around the issue.
__device__ __forceinline__ void mma_ktile_ts(uint32_t d_tm, uint32_t a_tm, uint32_t lo, uint32_t hi, uint32_t idesc,
                                             uint32_t accumulate, uint32_t empty_bar) {
  asm volatile(
      "{\n\t.reg .pred pe, pa, pt;\n\t"
      ".reg .b32 l1, l2, l3, a1, a2, a3;\n\t"
      ".reg .b64 d0, d1, d2, d3;\n\t"
      "elect.sync _|pe, 0xffffffff;\n\t"
      "setp.ne.b32 pa, %4, 0;\n\t"
      "setp.eq.b32 pt, 0, 0;\n\t"
      "add.u32 l1, %2, 2;\n\t"
      "add.u32 l2, %2, 4;\n\t"
      "add.u32 l3, %2, 6;\n\t"
      "add.u32 a1, %1, 8;\n\t"
      "add.u32 a2, %1, 16;\n\t"
      "add.u32 a3, %1, 24;\n\t"
      "mov.b64 d0, {%2, %3};\n\t"
      "mov.b64 d1, {l1, %3};\n\t"
      "mov.b64 d2, {l2, %3};\n\t"
      "mov.b64 d3, {l3, %3};\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], d0, %5, pa;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], d1, %5, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], d2, %5, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], d3, %5, pt;\n\t"
      "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}" ::"r"(d_tm),
      "r"(a_tm), "r"(lo), "r"(hi), "r"(accumulate), "r"(idesc), "r"(empty_bar)
      : "memory");
}

// Same k-tile with compile-time TMEM operand addresses (A = kA.., D = d_tm)
// and the X descriptor low word in a register: the stage index of the
// caller is a template constant, so the only runtime operands are the
// descriptor base, the accumulate flag and the barrier.
template <uint32_t kA>
__device__ __forceinline__ void mma_ktile_ts_imm(uint32_t d_tm, uint32_t lo, uint32_t hi, uint32_t idesc,
                                                 uint32_t accumulate, uint32_t empty_bar) {
  asm volatile(
      "{\n\t.reg .pred pe, pa, pt;\n\t"
      ".reg .b32 l1, l2, l3;\n\t"
      ".reg .b64 d0, d1, d2, d3;\n\t"
      "elect.sync _|pe, 0xffffffff;\n\t"
      "setp.ne.b32 pa, %3, 0;\n\t"
      "setp.eq.b32 pt, 0, 0;\n\t"
      "add.u32 l1, %1, 2;\n\t"
      "add.u32 l2, %1, 4;\n\t"
      "add.u32 l3, %1, 6;\n\t"
      "mov.b64 d0, {%1, %2};\n\t"
      "mov.b64 d1, {l1, %2};\n\t"
      "mov.b64 d2, {l2, %2};\n\t"
      "mov.b64 d3, {l3, %2};\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], d0, %4, pa;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], d1, %4, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], d2, %4, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], d3, %4, pt;\n\t"
      "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(d_tm),
      "r"(lo), "r"(hi), "r"(accumulate), "r"(idesc), "r"(empty_bar), "r"(kA), "r"(kA + 8), "r"(kA + 16),
      "r"(kA + 24)
      : "memory");
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> f32, A and B K-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t m, uint32_t n) {
  return (1u << 4)              // D format f32
         | (1u << 7)            // A bf16
         | (1u << 10)           // B bf16
         | ((n >> 3) << 17)     // N / 8
         | ((m >> 4) << 24);    // M / 16
}

}  // namespace salr
