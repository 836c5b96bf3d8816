// K2: varlen block-pair attention backward (dK, dV) on sm_100a (tcgen05 + TMEM + TMA).
//
// Work item = one 128-row KV block of one KV chunk (local or received) for one KV
// head.  The CTA streams every (Q chunk, 128-row Q block, q-head of the GQA group)
// that attends to it; dK/dV accumulate in TMEM and are written once (no atomics).
// dQ is produced by the query-stationary kernel in attn_dq_sm100.cuh: reducing a
// fp32 dQ partial per tile from here measured ~9 B/clk/SM of reduction throughput on
// B200 (TMA reduce-add and red.global alike), 2.3x the tile's tensor time.
//
// Per Q tile j (128 query rows of one q head):
//   S^T  = K  Q_j^T   M128 N128 K128 (SS)  -> TMEM S  [0,128)    fp32
//   dP^T = V  dO_j^T  M128 N128 K128 (SS)  -> TMEM dP [128,256)  fp32
//   softmax (thread == kv row; warpgroup w owns q columns [32w, 32w+32)):
//     phase 1: P^T = exp2(S^T*c - lse2[q])           -> bf16, in place over its own S columns
//     phase 2: dS^T = P^T (dP^T - delta[q])           -> bf16, in place over its own dP columns
//   dV  += P^T  dO_j  M128 N128 K128 (TS, A = P^T from TMEM)  -> TMEM dV [256,384)
//   dK  += dS^T Q_j   M128 N128 K128 (TS, A = dS^T from TMEM) -> TMEM dK [384,512)
// N=128 keeps the SS MMAs off the shared-memory operand limit (N=64 SS measured 48 vs 32
// cycles per instruction), and writing P/dS in place frees the TMEM a second S/dP buffer
// would need.  Issue order  dV(j), S(j+1), dK(j), dP(j+1):  the tensor pipe is in order, so
// S(j+1) cannot overwrite P(j) before dV(j) read it, nor dP(j+1) dS(j) before dK(j); and
// phase 1 of tile j+1 (the exp work) overlaps dK(j)/dP(j+1), phase 2 of tile j overlaps
// dV(j)/S(j+1).
// Operand rings: Q is held from S(j) to dK(j), dO from dP(j) to phase 2 of tile j (its slot
// carries delta), so Q gets three slots and dO two (227 KB of shared memory, exactly); lse2
// travels with the Q slot.  Phase 1 keeps P as the same bf16 pairs the dV MMA consumes.
// Warps: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-19 four softmax warpgroups, which
//        also drain dK/dV at the end of each item (four warps per SMSP hide the exp
//        phase's dependency latency; with two it ran at ~40% issue efficiency).
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

#ifndef FCPB_BWD_POLY
#define FCPB_BWD_POLY 1
#endif

namespace fcpb {
namespace bwd {

#ifdef FCPB_TRACE
// Debug timeline of CTA 0: [event][tile] clock64 stamps (see scripts/trace_bwd.py).
constexpr int kTraceTiles = 256;
enum TraceEv { kTrQIssue, kTrQGot, kTrSIssue, kTrPGot, kTrDvIssue, kTrDsGot, kTrDkIssue,
               kTrSGot, kTrPArrive, kTrDpGot, kTrDsArrive, kTrSLd, kTrPSt, kTrDpLd, kTrDsSt, kTrEvents };
__device__ unsigned long long g_trace[kTrEvents * kTraceTiles];
#define FCPB_TR(ev, j) do { if (blockIdx.x == 0 && (j) < kTraceTiles && (threadIdx.x & 31) == 0 && \
    ((ev) < kTrSGot ? true : threadIdx.x == 128)) \
    g_trace[(ev) * kTraceTiles + (j)] = clock64(); } while (0)
#else
#define FCPB_TR(ev, j) do {} while (0)
#endif

constexpr int kD = 128;
constexpr int kBK = 128;                        // kv rows per item
constexpr int kBQ = 128;                        // q rows per tile
constexpr int kKVBytes = kBK * kD * 2;          // 32 KB (two 16 KB SW128 panels of 64 d)
constexpr int kKVPanel = kKVBytes / 2;
constexpr int kQBytes = kBQ * kD * 2;           // 32 KB (two 16 KB panels)
constexpr int kQPanel = kQBytes / 2;
constexpr int kQSlots = 3;                      // Q ring depth (Q(j) is held until dK(j))
constexpr int kDoSlots = 2;                     // dO ring depth (dO(j) is freed with Q(j))
constexpr int kSoftmaxWGs = 4;
constexpr int kCols = kBQ / kSoftmaxWGs;        // q columns per softmax warpgroup
constexpr int kThreads = 128 * (1 + kSoftmaxWGs);
constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 384;
// Stacked tails (Params::stack_tails, GQA group even): the last Q block of a Q reference with
// at most 64 valid rows is one 128-column tile for TWO q-heads of the group -- columns 0-63
// are head gq's rows, 64-127 head gq+1's -- so dV and dK (summed over the group's heads
// anyway) take both in one pass.  Its dS^T tile goes to head gq's slot; the dQ GEMM reads it
// as 128 stacked rows (attn_dqg_sm100.cuh).
constexpr int kStackRows = 64;
// Register budget: 640 threads x 96 (the __launch_bounds__ allocation); the control and
// softmax warpgroups both fit in it, so no setmaxnreg split is needed.
constexpr uint32_t kRegsLaunch = 96;

// TMEM column of the bf16 A-operand chunk kk (16 q columns = 8 TMEM columns) of P^T / dS^T:
// warpgroup w keeps its 32 columns in the first 16 TMEM columns of its own S / dP slice.
FCPB_DEV constexpr uint32_t a_col(uint32_t base, int kk) {
  return base + static_cast<uint32_t>((kk >> 1) * kCols + (kk & 1) * 8);
}

// Position in a ring of N slots: slot index and the parity of the current lap.
template <int N>
struct RingPos {
  uint32_t slot = 0, phase = 0;
  FCPB_DEV void next() {
    if (++slot == N) { slot = 0; phase ^= 1; }
  }
};

struct KvSeg { int32_t kv_off, kv_len, flags, q_begin, q_end, pad_; };
struct QRef { int32_t q_off, q_len, diag, kv_limit; };   // kv_limit 0: every KV row visible
struct Item { int32_t kvseg, nblock; };

struct Smem {
  uint8_t k[kKVBytes];
  uint8_t v[kKVBytes];
  uint8_t q[kQSlots][kQBytes];
  uint8_t dout[kDoSlots][kQBytes];
  float lse2[kQSlots][kBQ];         // -lse * log2(e) (phase 1; travels with the Q slot)
  float delta[kDoSlots][kBQ];       // -delta (phase 2; travels with the dO slot)
  uint64_t kv_full, kv_empty;
  uint64_t q_full[kQSlots], q_empty[kQSlots];
  uint64_t do_full[kDoSlots], do_empty[kDoSlots];
  uint64_t s_full, dp_full, p_half, p_full, ds_full;
  uint64_t acc_full, acc_free;
  SchedRing sched;
  uint32_t tmem_base;
};

struct Params {
  int* sched_counter;      // dynamic tile scheduler (zeroed before launch)
  const KvSeg* kvsegs;
  const QRef* qrefs;
  const Item* items;
  int32_t num_items;
  int32_t num_q_heads, num_kv_heads;
  int32_t head_major;
  int32_t hm_lead;         // head_major: items run heads-adjacent before the head-major rest
  float scale;            // softmax scale
  float scale_log2;       // scale * log2(e)
  const float* lse2_t;    // [Hq, t_pad] -lse * log2(e)
  const float* delta_t;   // [Hq, t_pad] -delta
  int64_t t_pad;
  int32_t q_tokens;
  float* dk;              // local  [Tkv, Hkv, D] fp32
  float* dv;
  float* dk_recv;         // recv   [Tr, Hkv, D] fp32
  float* dv_recv;
  __nv_bfloat16* dk_out;  // optional final bf16 [Tkv, Hkv, D] for local segments
  __nv_bfloat16* dv_out;
  __nv_bfloat16* ds_out;  // optional dS^T tiles [pairs * Hq][128 q / 8][128 kv][8 q] for the dQ GEMM
  const int32_t* pair_base;  // per item: first (kv block, q block) pair id (worklist.build_ds_tiles)
  int32_t stack_tails;     // stacked tails (see kStackRows); requires an even GQA group
};

// Grid index -> (item, kv head).  head_major: neighbouring CTAs run neighbouring items of
// one head (they stream the same Q/dO tiles); else the heads of one item.
FCPB_DEV int item_of(int g, const Params& p) {
  int it, h;
  grid_map(g, p.num_items, p.num_kv_heads, p.head_major, p.hm_lead, it, h);
  return it;
}
FCPB_DEV int head_of(int g, const Params& p) {
  int it, h;
  grid_map(g, p.num_items, p.num_kv_heads, p.head_major, p.hm_lead, it, h);
  return h;
}

// Q blocks [q_first_block, q_end_block) of `qr` see KV block `nb` (128 rows): diagonal ->
// mb >= nb; a reference that sees only a prefix of the segment (kv_limit > 0, a received
// group's visible chunks) has none at or past it.
FCPB_DEV int q_first_block(const QRef& qr, int nb) { return qr.diag ? nb : 0; }
FCPB_DEV int q_end_block(const QRef& qr, int nb) {
  return (qr.kv_limit == 0 || nb * kBK < qr.kv_limit) ? (qr.q_len + kBQ - 1) / kBQ
                                                      : q_first_block(qr, nb);
}
// Is Q block mb of `qr` a stacked tail (two q-heads per tile)?
FCPB_DEV bool stacked_block(const QRef& qr, int mb, int stack) {
  return stack && qr.q_len - mb * kBQ <= kStackRows;
}
// (Q block, q-head) tiles of `qr` against KV block nb.
FCPB_DEV int qref_tiles(const QRef& qr, int nb, int group, int stack) {
  const int b0 = q_first_block(qr, nb), b1 = q_end_block(qr, nb);
  if (b1 <= b0) return 0;
  return (b1 - b0) * group - (stacked_block(qr, b1 - 1, stack) ? group / 2 : 0);
}

// 4-byte async copy with zero fill when !valid; completion tracked by an mbarrier.
FCPB_DEV void cp_async_4(void* smem_dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
               ::"r"(smem_u32(smem_dst)), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
FCPB_DEV void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

FCPB_DEV float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// Phase 1, 32 q columns of one kv row:  P = exp2(S*c + nlse2[q])  -> bf16 pairs in pk (kept
// for phase 2; the dV MMA consumes the same bf16 P) and stored at t_p.
// kMask: ragged kv row / ragged q / causal diagonal.
// Split P arrival: after its first 16 q columns every softmax thread stores them (8 TMEM
// columns) and arrives on p_half, so the MMA warp issues the dV K steps of those columns
// (kk = 0, 2, 4, 6 across the four warpgroups) while the second 16 are exponentiated.
#ifndef FCPB_BWD_PSPLIT
#define FCPB_BWD_PSPLIT 1
#endif
constexpr bool kPSplit = FCPB_BWD_PSPLIT != 0;
#ifndef FCPB_BWD_DS_LATE
#define FCPB_BWD_DS_LATE 1
#endif
constexpr bool kDsLate = FCPB_BWD_DS_LATE != 0;

template <bool kMask>
FCPB_DEV void p_chunk(const uint32_t (&s)[32], uint32_t l2, float sl2, uint32_t (&pk)[16], uint32_t t_p,
                      bool kv_live, int col0, int q_valid, int shift, uint64_t* p_half) {
  const float2 c2 = make_float2(sl2, sl2);
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8) {
    if (kPSplit && c8 == 2) {
      tmem_st8(t_p, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_half);
    }
    const float4 la = lds128(l2 + c8 * 32), lb = lds128(l2 + c8 * 32 + 16);
    const float2 nl[4] = {make_float2(la.x, la.y), make_float2(la.z, la.w),
                          make_float2(lb.x, lb.y), make_float2(lb.z, lb.w)};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = c8 * 8 + 2 * u;
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), c2, nl[u]);
      // Phase 1 is MUFU-bound (2 warps x 64 ex2 per SMSP per tile): every other pair goes
      // to the FMA pipe (FA4-style), which measured-balances MUFU time against issue slots.
      float p0, p1;
      // poly pairs per 4: FCPB_BWD_POLY (0..3); cycles on C2 with four softmax warpgroups:
      // 0: 13.50M, 1: 13.06M, 2: 13.37M, 3: 14.24M
      const bool use_poly = FCPB_BWD_POLY == 0 ? false : FCPB_BWD_POLY == 1 ? (u & 3) == 3
                            : FCPB_BWD_POLY == 2 ? (u & 1) != 0 : (u & 3) != 0;
      if (use_poly) {
        const float2 e = ex2_poly2(x);
        p0 = e.x;
        p1 = e.y;
      } else {
        p0 = ex2(x.x);
        p1 = ex2(x.y);
      }
      if (kMask) {
        const int col = col0 + i;
        p0 = (kv_live && col < q_valid && col >= shift) ? p0 : 0.f;
        p1 = (kv_live && col + 1 < q_valid && col + 1 >= shift) ? p1 : 0.f;
      }
      pk[c8 * 4 + u] = pack_bf16(p0, p1);
    }
  }
  if (kPSplit) tmem_st8(t_p + 8, pk + 8);
  else tmem_st16(t_p, pk);
}

// Phase 2, 32 q columns:  dS = P (dP + ndelta[q])  -> bf16 pairs at t_ds and in dk (the caller
// streams them into the materialised dS^T tile for the dQ GEMM after releasing ds_full).
FCPB_DEV void ds_chunk(const uint32_t (&dp)[32], uint32_t dl, const uint32_t (&pk)[16], uint32_t t_ds,
                       uint32_t (&dk)[16]) {
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8) {
    const float4 da = lds128(dl + c8 * 32), db = lds128(dl + c8 * 32 + 16);
    const float2 nd[4] = {make_float2(da.x, da.y), make_float2(da.z, da.w),
                          make_float2(db.x, db.y), make_float2(db.z, db.w)};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = c8 * 8 + 2 * u;
      const uint32_t pp = pk[c8 * 4 + u];     // bf16 pair: low half = column i
      const float2 dd = __fmul2_rn(
          make_float2(__uint_as_float(pp << 16), __uint_as_float(pp & 0xffff0000u)),
          __fadd2_rn(make_float2(__uint_as_float(dp[i]), __uint_as_float(dp[i + 1])), nd[u]));
      dk[c8 * 4 + u] = pack_bf16(dd.x, dd.y);
    }
  }
  tmem_st16(t_ds, dk);
}
// The 64 bytes of this thread's dS^T row into the tile, layout [q/8][kv][8 q]: chunk i at
// gdst[i * 128].  Streaming stores (keep L2 for the Q/dO stream), issued after ds_full is
// released: 32 KB per tile is ~1,100 cycles of one SM's share of HBM write bandwidth, and a
// full store queue stalling the warp before its arrival put it on the dK chain.
FCPB_DEV void ds_store(uint4* gdst, const uint32_t (&dk)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    st_global_cs(gdst + i * kBK, make_uint4(dk[4 * i], dk[4 * i + 1], dk[4 * i + 2], dk[4 * i + 3]));
}

__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q,      // bf16 [Tq,Hq,D], box (64,1,128)
                const __grid_constant__ CUtensorMap tm_do,     // bf16 [Tq,Hq,D], box (64,1,128)
                const __grid_constant__ CUtensorMap tm_q64,    // box (64,1,64): stacked tails
                const __grid_constant__ CUtensorMap tm_do64,
                const __grid_constant__ CUtensorMap tm_k,      // bf16 [Tkv,Hkv,D], box (64,1,128)
                const __grid_constant__ CUtensorMap tm_v,
                const __grid_constant__ CUtensorMap tm_k_recv,
                const __grid_constant__ CUtensorMap tm_v_recv,
                const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (reinterpret_cast<uint8_t*>(&sm) + sizeof(Smem) > smem_raw + dyn) __trap();
  }
  const uint32_t warp = warp_id();
  const int group = p.num_q_heads / p.num_kv_heads;
  const int total = p.num_items * p.num_kv_heads;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_q64);
    tma_prefetch_desc(&tm_do64);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_k_recv);
    tma_prefetch_desc(&tm_v_recv);
  }
  if (warp == 1 && elect_one()) {
    mbar_init(&sm.kv_full, 1);
    mbar_init(&sm.kv_empty, 1);
    for (int s = 0; s < kQSlots; ++s) {
      mbar_init(&sm.q_full[s], 1 + 32);   // TMA expect_tx arrive + 32 cp.async (lse2) arrives
      mbar_init(&sm.q_empty[s], 1);
    }
    for (int s = 0; s < kDoSlots; ++s) {
      mbar_init(&sm.do_full[s], 1 + 32);  // TMA expect_tx arrive + 32 cp.async (delta) arrives
      mbar_init(&sm.do_empty[s], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.dp_full, 1);
    mbar_init(&sm.p_half, 128 * kSoftmaxWGs);
    mbar_init(&sm.p_full, 128 * kSoftmaxWGs);
    mbar_init(&sm.ds_full, 128 * kSoftmaxWGs);
    mbar_init(&sm.acc_full, 1);
    mbar_init(&sm.acc_free, 128 * kSoftmaxWGs);
    sched_init(sm.sched, 1 + 4 * kSoftmaxWGs);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (all lanes:
      // lane 0 issues the TMA tiles, every lane copies 4 lse2 + 4 delta values with cp.async)
      const uint32_t lane = lane_id();
      const uint64_t keep = policy_evict_last();
      uint32_t kv_phase = 0;
      RingPos<kQSlots> qr_;
      RingPos<kDoSlots> dr_;
      int ptile = 0;
      SchedCursor sc;
      for (int g; (g = __shfl_sync(0xffffffffu, lane == 0 ? sched_produce(sm.sched, sc, p.sched_counter) : 0, 0)) < total;) {
        const Item it = p.items[item_of(g, p)];
        const int kvh = head_of(g, p);
        const KvSeg ks = p.kvsegs[it.kvseg];
        const bool recv = ks.flags & FCPB_KV_RECV;
        const int krow = ks.kv_off + it.nblock * kBK;
        bool kv_issued = false;
        auto issue_kv = [&]() {
          mbar_wait(&sm.kv_empty, kv_phase ^ 1);
          kv_phase ^= 1;
          if (lane == 0) {
            mbar_arrive_expect_tx(&sm.kv_full, 2 * kKVBytes);
            for (int half = 0; half < 2; ++half) {
              tma_load_3d(&sm.k[half * kKVPanel], recv ? &tm_k_recv : &tm_k, &sm.kv_full,
                          half * 64, kvh, krow);
              tma_load_3d(&sm.v[half * kKVPanel], recv ? &tm_v_recv : &tm_v, &sm.kv_full,
                          half * 64, kvh, krow);
            }
          }
          kv_issued = true;
        };
        for (int r = ks.q_begin; r < ks.q_end; ++r) {
          const QRef qr = p.qrefs[r];
          for (int mb = q_first_block(qr, it.nblock); mb < q_end_block(qr, it.nblock); ++mb) {
            const int qrow = qr.q_off + mb * kBQ;
            const bool stk = stacked_block(qr, mb, p.stack_tails);
            for (int gq = 0; gq < group; gq += stk ? 2 : 1) {
              const int h = kvh * group + gq;
              const uint32_t qs = qr_.slot, ds = dr_.slot;
              // stacked: 64-row boxes of heads h and h+1 fill rows 0-63 and 64-127 of each
              // 64-column panel (8 KB apart, whole 1 KB swizzle atoms)
              auto load_tile = [&](uint8_t* dst, const CUtensorMap* m, const CUtensorMap* m64, uint64_t* bar) {
                if (stk) {
                  for (int u = 0; u < 2; ++u)
                    for (int half = 0; half < 2; ++half)
                      tma_load_3d_hint(dst + half * kQPanel + u * (kQPanel / 2), m64, bar, half * 64,
                                       h + u, qrow, keep);
                } else {
                  for (int half = 0; half < 2; ++half)
                    tma_load_3d_hint(dst + half * kQPanel, m, bar, half * 64, h, qrow, keep);
                }
              };
              mbar_wait(&sm.q_empty[qs], qr_.phase ^ 1);
              if (lane == 0) {
                mbar_arrive_expect_tx(&sm.q_full[qs], kQBytes);
                load_tile(sm.q[qs], &tm_q, &tm_q64, &sm.q_full[qs]);
              }
              // column i: head h (+1 for stacked columns 64-127), query row qrow + (i mod 64)
#pragma unroll
              for (int u = 0; u < kBQ / 32; ++u) {
                const int i = lane + 32 * u;
                const int hi = stk ? h + (i >> 6) : h, ri = stk ? (i & (kStackRows - 1)) : i;
                const bool ok = qrow + ri < p.q_tokens;
                const float* src = p.lse2_t + static_cast<int64_t>(hi) * p.t_pad + qrow + ri;
                cp_async_4(&sm.lse2[qs][i], ok ? src : p.lse2_t, ok);
              }
              cp_async_arrive_noinc(&sm.q_full[qs]);
              // the first Q tile of an item goes out before K/V (they only wait on the ring)
              if (!kv_issued) issue_kv();
              mbar_wait(&sm.do_empty[ds], dr_.phase ^ 1);
              if (lane == 0) {
                mbar_arrive_expect_tx(&sm.do_full[ds], kQBytes);
                load_tile(sm.dout[ds], &tm_do, &tm_do64, &sm.do_full[ds]);
              }
#pragma unroll
              for (int u = 0; u < kBQ / 32; ++u) {
                const int i = lane + 32 * u;
                const int hi = stk ? h + (i >> 6) : h, ri = stk ? (i & (kStackRows - 1)) : i;
                const bool ok = qrow + ri < p.q_tokens;
                const float* src = p.delta_t + static_cast<int64_t>(hi) * p.t_pad + qrow + ri;
                cp_async_4(&sm.delta[ds][i], ok ? src : p.delta_t, ok);
              }
              cp_async_arrive_noinc(&sm.do_full[ds]);
              qr_.next();
              dr_.next();
              FCPB_TR(kTrQIssue, ptile); ++ptile;
            }
          }
        }
        if (!kv_issued) issue_kv();      // (items always have >= 1 tile; keeps phases paired)
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      const uint32_t id_sdp = idesc_bf16_f32(kBK, kBQ, false, false);  // S^T, dP^T
      const uint32_t id_acc = idesc_bf16_f32(kBK, kD, false, true);    // dV, dK (B MN-major)
      const uint32_t a_k = smem_u32(sm.k), a_v = smem_u32(sm.v);
      const bool leader = elect_one();
      uint32_t kv_phase = 0, acc_phase = 0;
      RingPos<kQSlots> qr_;
      RingPos<kDoSlots> dr_;
      uint32_t p_phase = 0, ds_phase = 0;
      uint32_t tile = 0;

      // S^T = K Q^T (b = Q slot) or dP^T = V dO^T (b = dO slot): K-major A and B.
      auto issue_kq = [&](uint32_t a_base, uint32_t b_base, uint32_t col, uint64_t* done) {
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * kKVPanel + (kk & 3) * 32;
            const uint32_t ob = (kk >> 2) * kQPanel + (kk & 3) * 32;
            mma_ss(tmem + col, smem_desc_sw128(a_base + oa, 16, 1024),
                   smem_desc_sw128(b_base + ob, 16, 1024), id_sdp, kk > 0);
          }
          mma_commit(done);
        }
        __syncwarp();
      };
      // dV += P^T dO  /  dK += dS^T Q:  A from TMEM, B = the [q, d] tile (MN-major).
      // kk_par: -1 all K steps; 0 / 1 the even / odd ones (first / second 16 columns of
      // every warpgroup's slice, the split-P halves)
      auto issue_acc = [&](uint32_t a_base, uint32_t b_base, uint32_t col, bool acc, uint64_t* done,
                           uint64_t* done2 = nullptr, int kk_par = -1) {
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kBQ / 16; ++kk)
            if (kk_par < 0 || (kk & 1) == kk_par)
              mma_ts(tmem + col, tmem + a_col(a_base, kk),
                     smem_desc_sw128(b_base + kk * 2048, kQPanel, 1024), id_acc, acc || kk > 0);
          if (done) mma_commit(done);
          if (done2) mma_commit(done2);
        }
        __syncwarp();
      };

      SchedCursor sc;
      for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
        const Item it = p.items[item_of(g, p)];
        const KvSeg ks = p.kvsegs[it.kvseg];
        int n = 0;
        for (int r = ks.q_begin; r < ks.q_end; ++r) {
          const QRef qr = p.qrefs[r];
          n += qref_tiles(qr, it.nblock, group, p.stack_tails);
        }
        mbar_wait(&sm.kv_full, kv_phase);
        kv_phase ^= 1;
        // prologue: S(0), dP(0).  The S/dP regions are free: the previous item's last
        // dV/dK were issued after its softmax finished with them (in-order pipe).
        mbar_wait(&sm.q_full[qr_.slot], qr_.phase);
        FCPB_TR(kTrQGot, (int)tile);
        tc_fence_after();
        issue_kq(a_k, smem_u32(sm.q[qr_.slot]), kColS, &sm.s_full);
        FCPB_TR(kTrSIssue, (int)tile);
        mbar_wait(&sm.do_full[dr_.slot], dr_.phase);
        tc_fence_after();
        issue_kq(a_v, smem_u32(sm.dout[dr_.slot]), kColDP, &sm.dp_full);
        for (int j = 0; j < n; ++j, ++tile) {
          const uint32_t qcur = qr_.slot, dcur = dr_.slot;
          qr_.next();
          dr_.next();
          if (kPSplit) {
            mbar_wait(&sm.p_half, p_phase);
            if (j == 0) {
              mbar_wait(&sm.acc_free, acc_phase ^ 1);   // epilogue drained the previous item
              acc_phase ^= 1;
            }
            tc_fence_after();
            issue_acc(kColS, smem_u32(sm.dout[dcur]), kColDV, j > 0, nullptr, nullptr, 0);
          }
          mbar_wait(&sm.p_full, p_phase);
          p_phase ^= 1;
          FCPB_TR(kTrPGot, (int)tile);
          if (!kPSplit && j == 0) {
            mbar_wait(&sm.acc_free, acc_phase ^ 1);   // epilogue drained the previous item
            acc_phase ^= 1;
          }
          tc_fence_after();
          // (split: kk = 0 of the tile was issued with the even half, so every odd step
          // accumulates; acc || kk > 0 holds for them)
          issue_acc(kColS, smem_u32(sm.dout[dcur]), kColDV, j > 0, nullptr, nullptr, kPSplit ? 1 : -1);
          FCPB_TR(kTrDvIssue, (int)tile);
          if (j + 1 < n) {
            mbar_wait(&sm.q_full[qr_.slot], qr_.phase);
            FCPB_TR(kTrQGot, (int)tile + 1);
            tc_fence_after();
            issue_kq(a_k, smem_u32(sm.q[qr_.slot]), kColS, &sm.s_full);
            FCPB_TR(kTrSIssue, (int)tile + 1);
          }
          mbar_wait(&sm.ds_full, ds_phase);
          ds_phase ^= 1;
          FCPB_TR(kTrDsGot, (int)tile);
          tc_fence_after();
          // dO(j) is freed with Q(j): phase 2 reads delta from the dO slot until ds_full(j)
          issue_acc(kColDP, smem_u32(sm.q[qcur]), kColDK, j > 0, &sm.q_empty[qcur], &sm.do_empty[dcur]);
          FCPB_TR(kTrDkIssue, (int)tile);
          if (j + 1 < n) {
            mbar_wait(&sm.do_full[dr_.slot], dr_.phase);
            tc_fence_after();
            issue_kq(a_v, smem_u32(sm.dout[dr_.slot]), kColDP, &sm.dp_full);
          }
        }
        if (leader) {
          mma_commit(&sm.acc_full);
          mma_commit(&sm.kv_empty);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax (thread == kv row)
    const int wg = (warp - 4) >> 2;                       // q columns [32 wg, 32 wg + 32)
    const int tid = ((warp & 3) << 5) + lane_id();        // kv row == TMEM lane
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_bits + kColS + wg * kCols;
    const uint32_t t_dp = tmem + lane_bits + kColDP + wg * kCols;
    const float sl2 = p.scale_log2;
    uint32_t s_phase = 0, dp_phase = 0, acc_phase = 0, tile = 0;
    RingPos<kQSlots> qr_;
    RingPos<kDoSlots> dr_;
    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      const Item it = p.items[item_of(g, p)];
      const int kvh = head_of(g, p);
      const KvSeg ks = p.kvsegs[it.kvseg];
      const int kv_row = it.nblock * kBK + tid;
      int pair = p.ds_out ? p.pair_base[item_of(g, p)] : 0;   // dS tiles: pair * Hq + q head
      for (int r = ks.q_begin; r < ks.q_end; ++r) {
        const QRef qr = p.qrefs[r];
        const int kv_end = qr.kv_limit ? min(qr.kv_limit, ks.kv_len) : ks.kv_len;
        const bool kv_live = kv_row < kv_end;
        const bool kv_full_tile = it.nblock * kBK + kBK <= kv_end;
        for (int mb = q_first_block(qr, it.nblock); mb < q_end_block(qr, it.nblock); ++mb, ++pair) {
          const int q_valid = qr.q_len - mb * kBQ;
          // diagonal: column c (q = 128 mb + c) sees kv row 128 nb + tid iff c >= shift
          const int shift0 = it.nblock * kBK - mb * kBQ;
          const bool plain = kv_full_tile && q_valid >= kBQ && (!qr.diag || shift0 + kBK - 1 <= 0);
          const int shift = qr.diag ? shift0 + tid : -(1 << 30);
          // stacked tail: two q-heads per tile (recomputed from q_valid where needed, which
          // keeps the per-tile loop inside its 96 registers)
          for (int gq = 0; gq < group; gq += (p.stack_tails && q_valid <= kStackRows) ? 2 : 1, ++tile) {
            uint32_t pr[kCols / 2];      // bf16 P pairs, phase 1 -> phase 2
            uint4* gdst = nullptr;
            if (p.ds_out) {
              const size_t tid_tile = static_cast<size_t>(pair) * p.num_q_heads + kvh * group + gq;
              // [q/8][kv][8 q]: a warp's 32 kv rows store 512 contiguous bytes per chunk,
              // and the tile is the no-swizzle MN-major canonical layout of the dQ GEMM's A
              gdst = reinterpret_cast<uint4*>(p.ds_out + tid_tile * (kBK * kBQ)) + (wg * 4) * kBK + tid;
            }
            mbar_wait(&sm.s_full, s_phase);
            s_phase ^= 1;
            FCPB_TR(kTrSGot, (int)tile);
            mbar_wait(&sm.q_full[qr_.slot], qr_.phase);   // lse2 of this tile landed
            tc_fence_after();
            const uint32_t l2 = smem_u32(&sm.lse2[qr_.slot][wg * kCols]);
            const uint32_t dl = smem_u32(&sm.delta[dr_.slot][wg * kCols]);
            // phase 1: P (bf16 lands over the first 16 of this warpgroup's S columns)
            {
              uint32_t sv[32];
              tmem_ld32(t_s, sv);
              tmem_wait_ld();
              FCPB_TR(kTrSLd, (int)tile);
              if (plain)
                p_chunk<false>(sv, l2, sl2, pr, t_s, true, 0, 0, 0, &sm.p_half);
              else
                p_chunk<true>(sv, l2, sl2, pr, t_s, kv_live,
                              // this warpgroup's first column as a query row of its head
                              ((p.stack_tails && q_valid <= kStackRows) ? (wg & 1) : wg) * kCols,
                              q_valid, shift, &sm.p_half);
            }
            FCPB_TR(kTrPSt, (int)tile);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_full);
            FCPB_TR(kTrPArrive, (int)tile);
            // phase 2: dS
            mbar_wait(&sm.dp_full, dp_phase);
            dp_phase ^= 1;
            mbar_wait(&sm.do_full[dr_.slot], dr_.phase);  // delta of this tile landed
            FCPB_TR(kTrDpGot, (int)tile);
            tc_fence_after();
            uint32_t dsk[16];
            {
              uint32_t dv[32];
              tmem_ld32(t_dp, dv);
              tmem_wait_ld();
              FCPB_TR(kTrDpLd, (int)tile);
              ds_chunk(dv, dl, pr, t_dp, dsk);
              FCPB_TR(kTrDsSt, (int)tile);
            }
            if (kDsLate) {
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&sm.ds_full);
              if (gdst) ds_store(gdst, dsk);
            } else {
              if (gdst) ds_store(gdst, dsk);
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&sm.ds_full);
            }
            FCPB_TR(kTrDsArrive, (int)tile);
            qr_.next();
            dr_.next();
          }
        }
      }
      // ---- dK/dV epilogue: this warpgroup's 32 d columns of its kv row
      mbar_wait(&sm.acc_full, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      {
        const bool recv = ks.flags & FCPB_KV_RECV;
        const bool kv_live = kv_row < ks.kv_len;
        const size_t row = (static_cast<size_t>(ks.kv_off + kv_row) * p.num_kv_heads + kvh) * kD + wg * 32;
        uint32_t a[32], bb[32];
        tmem_ld32(tmem + lane_bits + kColDK + wg * 32, a);
        tmem_ld32(tmem + lane_bits + kColDV + wg * 32, bb);
        tmem_wait_ld();
        if (kv_live && !recv && p.dk_out) {      // final bf16 (no partials come back)
          uint4* k4 = reinterpret_cast<uint4*>(p.dk_out + row);
          uint4* v4 = reinterpret_cast<uint4*>(p.dv_out + row);
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 wk, wv;
            wk.x = pack_bf16(__uint_as_float(a[i]) * p.scale, __uint_as_float(a[i + 1]) * p.scale);
            wk.y = pack_bf16(__uint_as_float(a[i + 2]) * p.scale, __uint_as_float(a[i + 3]) * p.scale);
            wk.z = pack_bf16(__uint_as_float(a[i + 4]) * p.scale, __uint_as_float(a[i + 5]) * p.scale);
            wk.w = pack_bf16(__uint_as_float(a[i + 6]) * p.scale, __uint_as_float(a[i + 7]) * p.scale);
            wv.x = pack_bf16(__uint_as_float(bb[i]), __uint_as_float(bb[i + 1]));
            wv.y = pack_bf16(__uint_as_float(bb[i + 2]), __uint_as_float(bb[i + 3]));
            wv.z = pack_bf16(__uint_as_float(bb[i + 4]), __uint_as_float(bb[i + 5]));
            wv.w = pack_bf16(__uint_as_float(bb[i + 6]), __uint_as_float(bb[i + 7]));
            k4[i / 8] = wk;
            v4[i / 8] = wv;
          }
        } else if (kv_live) {
          float* dkb = recv ? p.dk_recv : p.dk;
          float* dvb = recv ? p.dv_recv : p.dv;
          float4* k4 = reinterpret_cast<float4*>(dkb + row);
          float4* v4 = reinterpret_cast<float4*>(dvb + row);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            k4[i / 4] = make_float4(__uint_as_float(a[i]) * p.scale, __uint_as_float(a[i + 1]) * p.scale,
                                    __uint_as_float(a[i + 2]) * p.scale, __uint_as_float(a[i + 3]) * p.scale);
            v4[i / 4] = make_float4(__uint_as_float(bb[i]), __uint_as_float(bb[i + 1]),
                                    __uint_as_float(bb[i + 2]), __uint_as_float(bb[i + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.acc_free);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace bwd
}  // namespace fcpb
