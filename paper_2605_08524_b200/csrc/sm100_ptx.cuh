// Thin inline-PTX layer for sm_100a: mbarrier, TMA, tcgen05 (MMA / TMEM).
// Everything here compiles only for -gencode arch=compute_100a,code=sm_100a.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>

#define FCPB_DEV __device__ __forceinline__

namespace fcpb {

// ----------------------------------------------------------------------------- misc
FCPB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
FCPB_DEV uint32_t warp_id() { return threadIdx.x >> 5; }
FCPB_DEV uint32_t lane_id() { return threadIdx.x & 31; }
FCPB_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}
FCPB_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Per-warpgroup register budget (all 4 warps of the warpgroup must execute it).
template <uint32_t kRegs>
FCPB_DEV void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs)); }
template <uint32_t kRegs>
FCPB_DEV void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs)); }

// ----------------------------------------------------------------------------- mbarrier
FCPB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FCPB_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
FCPB_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
FCPB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}"
               ::"r"(smem_u32(bar)) : "memory");
}
FCPB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
FCPB_DEV bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
#ifndef FCPB_TRYWAIT_NS
#define FCPB_TRYWAIT_NS 0x989680u
#endif
// try_wait without a suspend-time hint lowers to SYNCS.PHASECHK.TRYWAIT (the hardware wait
// with its own short limit, then YIELD); with a hint it lowers to PHASECHK + NANOSLEEP.SYNCS,
// whose wake-up sits on every producer->consumer hand-off of the tile chains.  ncu cycles on
// C2 N=1 (r02, scripts/ab_cycles.sh): K1 5.82M -> 5.60M, K2 10.17M -> 9.63M, K2c unchanged;
// hints of 20 / 200 / 2,000 ns behave like the 10 ms one.
#ifndef FCPB_TRYWAIT_HINT
#define FCPB_TRYWAIT_HINT 0
#endif
FCPB_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if !FCPB_TRYWAIT_HINT
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(FCPB_TRYWAIT_NS)
      : "memory");
#endif
  return ok != 0;
}
FCPB_DEV uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifndef FCPB_WATCHDOG_NS
#define FCPB_WATCHDOG_NS 8000000000ull  // a pipeline stall this long is a bug: trap, don't hang
#endif
// printf in the (cold) watchdog path costs every kernel its spill-free register allocation:
// K2 spilled 88 B and ran 7.6% more cycles, K1 3.2%.  Build with -DFCPB_WATCHDOG_PRINT=1 to
// name the stuck barrier when debugging a hang; the trap itself is always there.
#ifndef FCPB_WATCHDOG_PRINT
#define FCPB_WATCHDOG_PRINT 0
#endif
// Spinning wait (no suspend): for a warp on the critical path (the MMA issuer), where the
// suspend/wake latency of try_wait would sit on the tile chain.
FCPB_DEV void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  if (mbar_test_wait(bar, parity)) return;
  const uint64_t t0 = global_timer_ns();
  uint32_t spins = 0;
  while (!mbar_test_wait(bar, parity)) {
    if ((++spins & 4095u) == 0 && global_timer_ns() - t0 > FCPB_WATCHDOG_NS) {
#if FCPB_WATCHDOG_PRINT
      printf("fcpb watchdog: block %d thread %d stuck on mbarrier smem+0x%x parity %u\n",
             blockIdx.x, threadIdx.x, smem_u32(bar), parity);
#endif
      __trap();
    }
  }
}
FCPB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = global_timer_ns();
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & 1023u) == 0 && global_timer_ns() - t0 > FCPB_WATCHDOG_NS) {
#if FCPB_WATCHDOG_PRINT
      printf("fcpb watchdog: block %d thread %d stuck on mbarrier smem+0x%x parity %u\n",
             blockIdx.x, threadIdx.x, smem_u32(bar), parity);
#endif
      __trap();
    }
  }
}

// ----------------------------------------------------------------------------- TMA
FCPB_DEV void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 3-D tiled load: coordinates innermost first (d, head, token).
FCPB_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                          int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
FCPB_DEV void tma_load_3d_hint(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int32_t c0,
                               int32_t c1, int32_t c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
FCPB_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
FCPB_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ----------------------------------------------------------------------------- tcgen05: TMEM
template <uint32_t kCols>
FCPB_DEV void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst_smem)), "n"(kCols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
FCPB_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}
FCPB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FCPB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
FCPB_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
FCPB_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 32 consecutive columns: thread t of the warp gets lane (base_lane + t).
FCPB_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
FCPB_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
FCPB_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
        "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
        "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]),
        "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 8 consecutive 32-bit columns from r[base..base+7]
FCPB_DEV void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
        "r"(r[7])
      : "memory");
}
FCPB_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
        "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
        "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// ----------------------------------------------------------------------------- tcgen05: MMA
// Shared-memory matrix descriptor (sm_100 "version 1"), SWIZZLE_128B.
//   bits  0-13 start address >> 4      bits 16-29 leading byte offset >> 4
//   bits 32-45 stride byte offset >> 4 bits 46-47 version (=1)
//   bits 49-51 base offset (0: atoms are 1024-B aligned)   bits 61-63 layout (2 = SW128)
FCPB_DEV uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Same descriptor for the no-swizzle ("interleave") canonical layout: 8x16-byte core
// matrices.  For an MN-major operand stored [MN/8][K][8] (16-byte rows of 8 MN elements,
// consecutive K rows 16 B apart): LBO = stride between K groups of 8 rows, SBO = stride
// between MN groups of 8 elements.
FCPB_DEV uint64_t smem_desc_noswz(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;                                        // layout type 0: no swizzle
}

// 16-byte streaming store (evict-first in L2: written once, read once later).
FCPB_DEV void st_global_cs(uint4* dst, uint4 v) {
  asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};"
               ::"l"(dst), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// 1-D bulk copy global -> shared with an L2 cache-policy hint.
FCPB_DEV void bulk_load_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}

// 1-D bulk copy global -> shared, completion on an mbarrier (transaction bytes).
FCPB_DEV void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Instruction descriptor, kind::f16: bf16 x bf16 -> f32.
//   bits 4-5 c fmt (1=f32), 7-9 a fmt (1=bf16), 10-12 b fmt (1=bf16),
//   bit 15 a major (0=K,1=MN), bit 16 b major, bits 17-22 N>>3, bits 24-28 M>>4
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N, bool a_mn,
                                                      bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]
FCPB_DEV void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
FCPB_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05 async ops of this thread complete.
FCPB_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

// ----------------------------------------------------------------------------- dynamic scheduler
// Persistent CTAs take work items from a global counter (zeroed before the launch), so
// CTAs that start late -- e.g. while NCCL kernels hold SMs during the exchange -- simply
// take fewer items.  The producer warp fetches; consumer warps read the item index from
// a small smem ring.  Index >= total means "no more work".
constexpr int kSchedSlots = 4;
struct SchedRing {
  int32_t item[kSchedSlots];
  uint64_t full[kSchedSlots];
  uint64_t empty[kSchedSlots];
};
FCPB_DEV void sched_init(SchedRing& r, uint32_t consumer_warps) {
  for (int i = 0; i < kSchedSlots; ++i) {
    mbar_init(&r.full[i], 1);
    mbar_init(&r.empty[i], consumer_warps);
  }
}
struct SchedCursor {
  uint32_t slot = 0, phase = 0;
  FCPB_DEV void advance() {
    if (++slot == kSchedSlots) { slot = 0; phase ^= 1; }
  }
};
// producer (one thread): claim the next item and publish it
FCPB_DEV int sched_produce(SchedRing& r, SchedCursor& c, int* counter) {
  mbar_wait(&r.empty[c.slot], c.phase ^ 1);
  const int g = atomicAdd(counter, 1);
  r.item[c.slot] = g;
  mbar_arrive(&r.full[c.slot]);
  c.advance();
  return g;
}
// consumer (whole warp): read the next item, release the slot once per warp
FCPB_DEV int sched_consume(SchedRing& r, SchedCursor& c) {
  mbar_wait(&r.full[c.slot], c.phase);
  const int g = *reinterpret_cast<volatile int32_t*>(&r.item[c.slot]);
  __syncwarp();
  if (lane_id() == 0) mbar_arrive(&r.empty[c.slot]);
  c.advance();
  return g;
}

// ----------------------------------------------------------------------------- work order
// Grid index g -> (item, head) for `items` LPT-ordered items x `heads` heads.
// head_major == 0: the heads of an item are adjacent.  Otherwise the first `lead` items run
// heads-adjacent (every head's largest items start first, no late tail) and the remaining
// items run head-major (one head's operand stream at a time stays in L2).
FCPB_DEV void grid_map(int g, int items, int heads, int head_major, int lead, int& item, int& head) {
  const int k = head_major ? (lead < items ? lead : items) : items;
  if (g < k * heads) {
    item = g / heads;
    head = g % heads;
    return;
  }
  g -= k * heads;
  const int rest = items - k;
  item = k + g % rest;
  head = g / rest;
}

// ----------------------------------------------------------------------------- math
FCPB_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair on the FMA/ALU pipes (x <= 127) (FA4-style MUFU offload): x = j + f, j = rint(x)
// via the 1.5*2^23 magic add, 2^f on [-0.5, 0.5] by a degree-3 polynomial (max rel err
// 7.7e-5, far below the bf16 rounding of P), 2^j folded into the exponent bits.
FCPB_DEV float2 ex2_poly2(float2 x) {
  // clamp: 2^j is folded into q's exponent (q in [0.7, 1.42], exponent 126..127), so j must
  // stay >= -125 to remain a normal number; 2^-125 (masked entries) is numerically zero here.
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 q = __ffma2_rn(make_float2(0.055088766f, 0.055088766f), f,
                        make_float2(0.24260466f, 0.24260466f));
  q = __ffma2_rn(q, f, make_float2(0.6932763f, 0.6932763f));
  q = __ffma2_rn(q, f, make_float2(0.9999289f, 0.9999289f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}

FCPB_DEV float fmax3(float a, float b, float c) {   // FMNMX3 (sm_100)
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

FCPB_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace fcpb
