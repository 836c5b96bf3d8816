// K1: varlen block-pair attention forward on sm_100a (tcgen05 + TMEM + TMA).
//
// One persistent CTA per SM.  A work item is 128 query rows of one FCP segment
// (a Q chunk plus the ordered KV chunks it attends to in this launch) for a
// *pair* of query heads that share one KV head (GQA), so every K/V tile that
// TMA stages in shared memory feeds two Q tiles.
//
// Warp roles (12 warps):
//   w0      TMA producer: Q pair once per item, then K(j), V(j) into a 4-slot ring
//   w1      MMA issuer (one elected lane): S_h = Q_h K^T (SS), O_h += P_h V (TS)
//   w2      TMEM allocator (512 columns)
//   w3      idle
//   w4-7    softmax/epilogue for head 0 of the pair (thread == query row)
//   w8-11   softmax/epilogue for head 1 of the pair
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_h (bf16,
// 64 columns) overwrites the first half of S_h once S_h has been read.
// MMA order per KV tile j:  PV0(j), S0(j+1), PV1(j), S1(j+1): the tensor pipe
// runs one head's matmuls while the other head's warps do the softmax.
// Stacked tails (stack_tails, GQA group a multiple of 4): the last Q tile of a segment with
// at most 64 valid rows carries FOUR q-heads -- tile h holds the 64 rows of head 4k+2h in
// TMEM lanes 0-63 and those of head 4k+2h+1 in lanes 64-127 (all four share the KV head) --
// so a short Q run's ragged tail costs half a tile pair; the odd head pair of such an item
// is empty.  At N >= 2 about 5% of C2's forward tiles are such tails.
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

namespace fcpb {
namespace fwd {

#ifdef FCPB_TRACE
constexpr int kTraceTiles = 256;
enum FwdEv { kFwKGot, kFwS0Issue, kFwP0Got, kFwPv0Issue, kFwP1Got, kFwPv1Issue, kFwS0Got, kFwP0Arrive,
             kFwS1Got, kFwP1Arrive, kFwSLd0, kFwMax0, kFwExp0, kFwEvents };
__device__ unsigned long long g_trace[kFwEvents * kTraceTiles];
#define FCPB_FWTR(ev, j) do { if (blockIdx.x == 0 && (j) < kTraceTiles && (threadIdx.x & 31) == 0 && \
    ((ev) < kFwS0Got ? true : (threadIdx.x == 128 || threadIdx.x == 256))) \
    g_trace[(ev) * kTraceTiles + (j)] = clock64(); } while (0)
#else
#define FCPB_FWTR(ev, j) do {} while (0)
#endif

// Test hook: warp-level O-rescale events of the lazy (thresholded) softmax rescale, read
// through fcpb_debug_counters() so parity tests can prove the rescale path ran.  The branch
// is rare in practice (the row max must grow by > 2^8 in the exp2 domain), so the atomic is
// off the hot path.
__device__ unsigned long long g_rescales;

constexpr int kD = 128;          // head dim
constexpr int kBM = 128;         // query rows per tile
constexpr int kBN = 128;         // kv rows per tile
constexpr int kSlots = 4;        // K/V ring slots (each one K or one V tile)
constexpr int kTileBytes = kBN * kD * 2;        // 32 KB
constexpr int kHalfBytes = kTileBytes / 2;      // one 64-column swizzle panel
constexpr int kThreads = 384;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 384;

struct Smem {
  uint8_t q[2][kTileBytes];           // 64 KB, 1024-aligned panels
  uint8_t kv[kSlots][kTileBytes];     // 128 KB
  uint64_t q_full, q_empty;
  uint64_t kv_full[kSlots], kv_empty[kSlots];
  uint64_t s_full[2], p_part[2], p_full[2], o_full[2], o_empty[2];
  SchedRing sched;
  uint32_t tmem_base;
};

struct Params {
  int* sched_counter;      // dynamic tile scheduler (zeroed before launch)
  const FcpbSegment* segs;
  const FcpbKvRef* kvrefs;
  const FcpbItem* items;
  int32_t num_items;
  int32_t num_q_heads;
  int32_t num_kv_heads;
  int32_t head_major;    // grid index -> (item, head pair) mapping
  int32_t hm_lead;         // head_major: items run heads-adjacent before the head-major rest
  float scale_log2;      // softmax_scale * log2(e)
  float scale;           // softmax_scale
  __nv_bfloat16* o;      // [Tq, Hq, D]
  float* lse;            // [Tq, Hq]
  float* o_part;         // [P, Hq, D]
  float* lse_part;       // [P, Hq]
  int32_t stack_tails;   // tail tiles with <= 64 rows carry four q-heads (group % 4 == 0)
};

constexpr int kStackRows = 64;   // a stacked tile: 64 rows of each of two q-heads

// Does item `it` (128-row block of `seg`) run stacked?  The odd head pair of a stacked item
// is empty (its four heads ran under the even pair).
FCPB_DEV bool stacked(const Params& p, const FcpbSegment& seg, const FcpbItem& it) {
  return p.stack_tails && seg.q_len - it.mblock * kBM <= kStackRows;
}

FCPB_DEV int item_of(int g, int hp, const Params& p) {
  int it, h;
  grid_map(g, p.num_items, hp, p.head_major, p.hm_lead, it, h);
  return it;
}
FCPB_DEV int pair_of(int g, int hp, const Params& p) {
  int it, h;
  grid_map(g, p.num_items, hp, p.head_major, p.hm_lead, it, h);
  return h;
}

// Number of 128-row KV tiles a Q tile at m-block `mb` visits in `ref`.
FCPB_DEV int kv_tiles(const FcpbKvRef& ref, int mb) {
  int n = (ref.len + kBN - 1) / kBN;
  if (ref.flags & FCPB_KV_DIAG) n = min(n, mb + 1);
  return n;
}

#ifndef FCPB_FWD_POLY_PAIRS
#define FCPB_FWD_POLY_PAIRS 2    // exp2 pairs of every 8 on the FMA pipe (ncu C2 r02: 2 best)
#endif
constexpr int kPolyPairs = FCPB_FWD_POLY_PAIRS;

// Split P arrival (FA4-style): after the first kPSplit of the four 32-column chunks of P are
// in TMEM the softmax warps arrive on p_part, and the MMA warp issues those K steps of
// O += P V while the rest are packed and stored; p_full releases the rest.  The O rescale
// (rare) therefore happens before the exponentials.
#ifndef FCPB_FWD_PSPLIT
#define FCPB_FWD_PSPLIT 2    // ncu A/B on C2 (r02): 2 chunks best (0/1/3: +5% / +4% / +5%)
#endif
constexpr int kPSplit = FCPB_FWD_PSPLIT;
static_assert(kPSplit >= 0 && kPSplit < 4, "P split point in 32-column chunks");

// One row of a 128-column S tile, FA4 order: every exponential first, in place in s --
// P = exp2(s*sl2 + neg), pairs 8u+8-kPolyPairs..8u+7 by ex2_poly2 when kPoly (finite inputs
// only) -- then the bf16 pack and TMEM store per 32-column chunk (16 columns at t_s + 16c,
// over S columns already read), arriving on p_part after kPSplit chunks.  The caller sums the
// exponentials left in s after releasing P (row_sum).  ncu C2 (r02): 5.32M -> 5.23M cycles
// with 2 polynomial pairs, against inline sums and per-chunk stores with 1 pair.
template <bool kPoly>
FCPB_DEV void exp_row(float (&s)[kBN], float sl2, float neg, uint32_t t_s, uint64_t* p_part) {
#pragma unroll
  for (int i = 0; i < kBN; i += 2) {
    const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), make_float2(sl2, sl2), make_float2(neg, neg));
    float2 e;
    if (kPoly && ((i >> 1) & 7) >= 8 - kPolyPairs) e = ex2_poly2(x);
    else e = make_float2(ex2(x.x), ex2(x.y));
    s[i] = e.x;
    s[i + 1] = e.y;
  }
#pragma unroll
  for (int c = 0; c < kBN / 32; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]);
    tmem_st16(t_s + c * 16, pk);
    if (kPSplit > 0 && c + 1 == kPSplit) {
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_part);
    }
  }
}

// Sum of the 128 exponentials exp_row leaves in s, 4 independent chains.
FCPB_DEV float row_sum(const float (&s)[kBN]) {
  float2 a[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < kBN; i += 2) a[(i >> 1) & 3] = __fadd2_rn(a[(i >> 1) & 3], make_float2(s[i], s[i + 1]));
  const float2 b = __fadd2_rn(__fadd2_rn(a[0], a[1]), __fadd2_rn(a[2], a[3]));
  return b.x + b.y;
}

// setmaxnreg split: one producer/MMA warpgroup, two softmax warpgroups.  setmaxnreg.inc can
// only take registers the CTA was given at launch (384 threads x 168, the __launch_bounds__
// allocation), so the budgets must sum to at most 3 * kRegsLaunch.
constexpr uint32_t kRegsLaunch = 168, kRegsCtl = 104, kRegsSoftmax = 200;
static_assert(kRegsCtl + 2 * kRegsSoftmax <= 3 * kRegsLaunch,
              "setmaxnreg.inc would wait forever for registers that were never allocated");

__global__ void __launch_bounds__(kThreads, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_q64,   // Q with 64-row boxes (stacked tails)
                const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v,
                const __grid_constant__ CUtensorMap tm_k_recv,
                const __grid_constant__ CUtensorMap tm_v_recv,
                const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id();
  const int head_pairs = p.num_q_heads / 2;
  const int group = p.num_q_heads / p.num_kv_heads;
  const int total = p.num_items * head_pairs;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_q64);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_k_recv);
    tma_prefetch_desc(&tm_v_recv);
  }
  if (warp == 1 && elect_one()) {
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&sm.s_full[h], 1);
      mbar_init(&sm.p_part[h], 128);
      mbar_init(&sm.p_full[h], 128);
      mbar_init(&sm.o_full[h], 1);
      mbar_init(&sm.o_empty[h], 128);
    }
    sched_init(sm.sched, 1 + 8);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    // producer / MMA warpgroup: few registers, the rest go to the softmax warpgroups
    reg_dealloc<kRegsCtl>();
    if (warp == 0) {
      // ------------------------------------------------------------ TMA producer
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t q_phase = 0, slot = 0, slot_phase = 0;
        SchedCursor sc;
        for (int g; (g = sched_produce(sm.sched, sc, p.sched_counter)) < total;) {
          const FcpbItem it = p.items[item_of(g, head_pairs, p)];
          const int hp = pair_of(g, head_pairs, p);
          const FcpbSegment seg = p.segs[it.seg];
          const bool stk = stacked(p, seg, it);
          if (stk && (hp & 1)) continue;             // ran under the even pair
          const int h0 = 2 * hp;
          const int kvh = h0 / group;
          const int row0 = seg.q_off + it.mblock * kBM;
          mbar_wait(&sm.q_empty, q_phase ^ 1);
          q_phase ^= 1;
          mbar_arrive_expect_tx(&sm.q_full, 2 * kTileBytes);
          if (stk) {
            // tile h: rows 0-63 of head h0+2h, then rows 0-63 of head h0+2h+1 (64-row boxes;
            // 64 swizzled 128-byte rows = 8 KB, a whole number of 1 KB swizzle atoms)
            for (int h = 0; h < 2; ++h)
              for (int u = 0; u < 2; ++u)
                for (int half = 0; half < 2; ++half)
                  tma_load_3d(&sm.q[h][half * kHalfBytes + u * (kHalfBytes / 2)], &tm_q64, &sm.q_full,
                              half * 64, h0 + 2 * h + u, row0);
          } else {
            for (int h = 0; h < 2; ++h)
              for (int half = 0; half < 2; ++half)
                tma_load_3d(&sm.q[h][half * kHalfBytes], &tm_q, &sm.q_full, half * 64, h0 + h, row0);
          }
          for (int r = seg.kv_begin; r < seg.kv_end; ++r) {
            const FcpbKvRef ref = p.kvrefs[r];
            const bool recv = ref.flags & FCPB_KV_RECV;
            const CUtensorMap* mk = recv ? &tm_k_recv : &tm_k;
            const CUtensorMap* mv = recv ? &tm_v_recv : &tm_v;
            const int nt = kv_tiles(ref, it.mblock);
            for (int t = 0; t < nt; ++t) {
              const int krow = ref.off + t * kBN;
              for (int kv = 0; kv < 2; ++kv) {
                mbar_wait(&sm.kv_empty[slot], slot_phase ^ 1);
                mbar_arrive_expect_tx(&sm.kv_full[slot], kTileBytes);
                const CUtensorMap* m = kv ? mv : mk;
                for (int half = 0; half < 2; ++half)
                  tma_load_3d_hint(&sm.kv[slot][half * kHalfBytes], m, &sm.kv_full[slot], half * 64,
                                   kvh, krow, keep);
                if (++slot == kSlots) { slot = 0; slot_phase ^= 1; }
              }
            }
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t id_s = idesc_bf16_f32(kBM, kBN, false, false);
      const uint32_t id_o = idesc_bf16_f32(kBM, kD, false, true);
      const uint32_t q_addr0 = smem_u32(sm.q[0]), q_addr1 = smem_u32(sm.q[1]);
      // selects, not arrays: a runtime-indexed array would live in local memory
      auto q_addr = [&](int h) { return h ? q_addr1 : q_addr0; };
      auto col_s = [](int h) { return h ? kColS1 : kColS0; };
      auto col_o = [](int h) { return h ? kColO1 : kColO0; };
      uint32_t q_phase = 0, slot = 0, slot_phase = 0, p_phase = 0, oe_phase = 0;
      int trt = 0;   // trace tile counter
      const bool leader = elect_one();
      auto issue_s = [&](int h, uint32_t kslot) {
        if (leader) {
          const uint32_t kb = smem_u32(sm.kv[kslot]);
  #pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
            mma_ss(tmem + col_s(h), smem_desc_sw128(q_addr(h) + off, 16, 1024),
                   smem_desc_sw128(kb + off, 16, 1024), id_s, kk > 0);
          }
          mma_commit(&sm.s_full[h]);
        }
        __syncwarp();
      };
      // O_h += P_h V over K steps [kk0, kk1) (16 kv rows each)
      auto issue_pv = [&](int h, uint32_t vslot, bool acc, int kk0, int kk1) {
        if (leader) {
          const uint32_t vb = smem_u32(sm.kv[vslot]);
  #pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {
            if (kk < kk0 || kk >= kk1) continue;
            mma_ts(tmem + col_o(h), tmem + col_s(h) + kk * 8,
                   smem_desc_sw128(vb + kk * 2048, kHalfBytes, 1024), id_o, (acc || kk > 0));
          }
        }
        __syncwarp();
      };
      constexpr int kKkSplit = kPSplit * 2;     // K steps covered by the first P chunks
      // wait for P_h(j) (in two parts when split) and issue O_h += P_h V_j
      auto pv = [&](int h, uint32_t vslot, bool acc) {
        if (kPSplit > 0) {
          mbar_wait(&sm.p_part[h], p_phase);
          tc_fence_after();
          issue_pv(h, vslot, acc, 0, kKkSplit);
        }
        mbar_wait(&sm.p_full[h], p_phase);
        if (h == 0) FCPB_FWTR(kFwP0Got, trt); else FCPB_FWTR(kFwP1Got, trt);
        tc_fence_after();
        issue_pv(h, vslot, acc, kPSplit > 0 ? kKkSplit : 0, kBN / 16);
      };
      auto commit = [&](uint64_t* bar) {
        if (leader) mma_commit(bar);
        __syncwarp();
      };
      // Take the next ring position and wait until TMA has filled it.
      auto take_full = [&]() {
        const uint32_t cur = slot;
        mbar_wait(&sm.kv_full[cur], slot_phase);
        if (++slot == kSlots) { slot = 0; slot_phase ^= 1; }
        return cur;
      };

      SchedCursor sc;
      for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
        const FcpbItem it = p.items[item_of(g, head_pairs, p)];
        const FcpbSegment seg = p.segs[it.seg];
        if (stacked(p, seg, it) && (pair_of(g, head_pairs, p) & 1)) continue;
        int n = 0;
        for (int r = seg.kv_begin; r < seg.kv_end; ++r) n += kv_tiles(p.kvrefs[r], it.mblock);
        mbar_wait(&sm.q_full, q_phase);
        q_phase ^= 1;
        // O accumulators of the previous item must have been drained by the epilogue.
        mbar_wait(&sm.o_empty[0], oe_phase ^ 1);
        mbar_wait(&sm.o_empty[1], oe_phase ^ 1);
        oe_phase ^= 1;
        tc_fence_after();
        // K(0)
        const uint32_t ks = take_full();
        tc_fence_after();
        issue_s(0, ks);
        issue_s(1, ks);
        commit(&sm.kv_empty[ks]);
        if (n == 1) commit(&sm.q_empty);
        const bool resumed = seg.in_row > 0;      // O starts from an earlier wave's partial
        for (int j = 0; j < n; ++j) {
          const uint32_t vs = take_full();
          pv(0, vs, j > 0 || resumed);
          FCPB_FWTR(kFwPv0Issue, trt);
          if (j == n - 1) commit(&sm.o_full[0]);
          uint32_t ks2 = 0;
          if (j + 1 < n) {
            ks2 = take_full();
            FCPB_FWTR(kFwKGot, trt + 1);
            tc_fence_after();
            issue_s(0, ks2);
            FCPB_FWTR(kFwS0Issue, trt + 1);
          }
          pv(1, vs, j > 0 || resumed);
          FCPB_FWTR(kFwPv1Issue, trt);
          commit(&sm.kv_empty[vs]);
          if (j == n - 1) commit(&sm.o_full[1]);
          if (j + 1 < n) {
            issue_s(1, ks2);
            commit(&sm.kv_empty[ks2]);
            if (j + 2 == n) commit(&sm.q_empty);
          }
          p_phase ^= 1;
          ++trt;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    reg_alloc<kRegsSoftmax>();
    const int h = (warp - 4) >> 2;           // which head of the pair
    const int row = (warp & 3) * 32 + lane_id();
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_bits + (h ? kColS1 : kColS0);
    const uint32_t t_o = tmem + lane_bits + (h ? kColO1 : kColO0);
    uint32_t s_phase = 0, o_phase = 0;
    int trt = 0;
    const float sl2 = p.scale_log2;

    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      const FcpbItem it = p.items[item_of(g, head_pairs, p)];
      const int hp = pair_of(g, head_pairs, p);
      const FcpbSegment seg = p.segs[it.seg];
      const bool stk = stacked(p, seg, it);
      if (stk && (hp & 1)) continue;
      // this thread's query: head and row inside the 128-row block (stacked: lanes 64-127
      // hold the second head's rows 0-63)
      const int head = stk ? 2 * hp + 2 * h + (row >> 6) : 2 * hp + h;
      const int qr = stk ? (row & (kStackRows - 1)) : row;
      float m_run = -INFINITY, l_run = 0.f;
      bool first = true;
      if (seg.in_row > 0) {
        // Continue an earlier wave's (O, LSE) partial: O (normalised, fp32) into TMEM, the
        // running max at LSE / scale with l = 1, so exp((s - m) * scale) = exp(s * scale - LSE)
        // carries on exactly; the lazy rescale then applies to the loaded O.  The MMA warp's
        // first PV accumulates onto it (its p_full wait orders after these stores).
        const int qrow = it.mblock * kBM + qr;
        const bool live = qrow < seg.q_len;
        const size_t prow = static_cast<size_t>(seg.in_row - 1 + qrow) * p.num_q_heads + head;
        const float4* src = reinterpret_cast<const float4*>(p.o_part + prow * kD);
#pragma unroll 1
        for (int c = 0; c < kD / 16; ++c) {
          uint32_t v[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 x = live ? src[c * 4 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
            v[4 * i] = __float_as_uint(x.x);
            v[4 * i + 1] = __float_as_uint(x.y);
            v[4 * i + 2] = __float_as_uint(x.z);
            v[4 * i + 3] = __float_as_uint(x.w);
          }
          tmem_st16(t_o + c * 16, v);
        }
        tmem_wait_st();
        if (live) {
          m_run = p.lse_part[prow] / p.scale;
          l_run = 1.f;
        }
        first = false;
      }
      for (int r = seg.kv_begin; r < seg.kv_end; ++r) {
        const FcpbKvRef ref = p.kvrefs[r];
        const int nt = kv_tiles(ref, it.mblock);
        const bool diag = ref.flags & FCPB_KV_DIAG;
        for (int t = 0; t < nt; ++t) {
          mbar_wait(&sm.s_full[h], s_phase);
          s_phase ^= 1;
          if (h == 0) FCPB_FWTR(kFwS0Got, trt); else FCPB_FWTR(kFwS1Got, trt);
          tc_fence_after();
          float s[kBN];
          {
            // all four 32-column loads in flight before one wait: one load latency, not four
            // (-2% cycles against a wait per load)
            uint32_t v0[32], v1[32], v2[32], v3[32];
            tmem_ld32(t_s, v0);
            tmem_ld32(t_s + 32, v1);
            tmem_ld32(t_s + 64, v2);
            tmem_ld32(t_s + 96, v3);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              s[i] = __uint_as_float(v0[i]);
              s[32 + i] = __uint_as_float(v1[i]);
              s[64 + i] = __uint_as_float(v2[i]);
              s[96 + i] = __uint_as_float(v3[i]);
            }
          }
          if (h == 0) FCPB_FWTR(kFwSLd0, trt);
          // masking: ragged KV tail, causal diagonal (col <= row within the block)
          // (one unrolled loop for both: the kernel's code size sits near the instruction
          // cache's, so every unrolled 128-column loop counts)
          const int valid = ref.len - t * kBN;
          const int lim = (diag && t == it.mblock) ? qr + 1 : valid;
          if (lim < kBN) {
#pragma unroll
            for (int i = 0; i < kBN; ++i)
              if (i >= lim) s[i] = -INFINITY;
          }
          float mp[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) mp[i] = fmax3(m_run, s[2 * i], s[2 * i + 1]);
#pragma unroll
          for (int i = 16; i < kBN; i += 2) mp[(i >> 1) & 7] = fmax3(mp[(i >> 1) & 7], s[i], s[i + 1]);
          const float mx = fmax3(fmax3(mp[0], mp[1], mp[2]), fmax3(mp[3], mp[4], mp[5]),
                                 fmaxf(mp[6], mp[7]));
          // Lazy rescale (FA4): keep exponentiating against the running reference max
          // until the row max grows by more than 2^8 in the exp2 domain, so O is
          // rescaled in TMEM only rarely.  P <= 2^8 stays exact enough in bf16/fp32.
          if (h == 0) FCPB_FWTR(kFwMax0, trt);
          float m_use;
          if (m_run == -INFINITY) m_use = (mx == -INFINITY) ? 0.f : mx;
          else m_use = ((mx - m_run) * sl2 > 8.f) ? mx : m_run;
          const float neg = -m_use * sl2;
          const float alpha = (m_run == -INFINITY) ? 0.f : ex2((m_run - m_use) * sl2);
          // tcgen05.ld/st are .sync.aligned: the rescale decision must be warp-uniform.  It runs
          // before the exponentials, so the first P chunks can release their PV K steps.
          if (!first && __any_sync(0xffffffffu, alpha != 1.f)) {
            // O_h(j-1) is final here: S_h(j) completed after PV_h(j-1) in the tensor pipe.
            if (lane_id() == 0) atomicAdd(&g_rescales, 1ull);
            // 16 columns at a time: the 128 scores of the row are live here
#pragma unroll 1
            for (int c = 0; c < kD / 16; ++c) {
              uint32_t v[16];
              tmem_ld16(t_o + c * 16, v);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
              tmem_st16(t_o + c * 16, v);
            }
          }
          // P (bf16 pairs) overwrites the first 64 columns of S, 16 columns per 32 scores.
          // Unmasked tiles (finite scores, x <= 8) send kPolyPairs of every 8 pairs to the
          // FMA pipe (FA4-style).  Masked tiles keep exact zeros from MUFU ex2(-inf).  The
          // choice is CTA-uniform.
          const bool poly = kPolyPairs > 0 && !(diag && t == it.mblock) && valid >= kBN;
          if (poly) exp_row<true>(s, sl2, neg, t_s, &sm.p_part[h]);
          else exp_row<false>(s, sl2, neg, t_s, &sm.p_part[h]);
          if (h == 0) FCPB_FWTR(kFwExp0, trt);
          m_run = (m_run == -INFINITY && mx == -INFINITY) ? -INFINITY : m_use;
          first = false;
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&sm.p_full[h]);
          if (h == 0) FCPB_FWTR(kFwP0Arrive, trt); else FCPB_FWTR(kFwP1Arrive, trt);
          l_run = l_run * alpha + row_sum(s);
          ++trt;
        }
      }
      // -------------------------------------------------------- epilogue
      mbar_wait(&sm.o_full[h], o_phase);
      o_phase ^= 1;
      tc_fence_after();
      const int qrow = it.mblock * kBM + qr;
      const bool live = qrow < seg.q_len;
      const float inv_l = (l_run > 0.f) ? 1.f / l_run : 0.f;
      const float lse = (l_run > 0.f) ? (m_run == -INFINITY ? 0.f : m_run) * p.scale + logf(l_run)
                                      : -INFINITY;
      if (seg.out_row < 0) {
        __nv_bfloat16* dst = p.o + (static_cast<size_t>(seg.q_off + qrow) * p.num_q_heads + head) * kD;
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_o + c * 32, v);
          tmem_wait_ld();
          if (live) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 w;
              w.x = pack_bf16(__uint_as_float(v[i + 0]) * inv_l, __uint_as_float(v[i + 1]) * inv_l);
              w.y = pack_bf16(__uint_as_float(v[i + 2]) * inv_l, __uint_as_float(v[i + 3]) * inv_l);
              w.z = pack_bf16(__uint_as_float(v[i + 4]) * inv_l, __uint_as_float(v[i + 5]) * inv_l);
              w.w = pack_bf16(__uint_as_float(v[i + 6]) * inv_l, __uint_as_float(v[i + 7]) * inv_l);
              d4[i / 8] = w;
            }
          }
        }
        if (live) p.lse[static_cast<size_t>(seg.q_off + qrow) * p.num_q_heads + head] = lse;
      } else {
        float* dst = p.o_part + (static_cast<size_t>(seg.out_row + qrow) * p.num_q_heads + head) * kD;
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_o + c * 32, v);
          tmem_wait_ld();
          if (live) {
            float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              d4[i / 4] = make_float4(__uint_as_float(v[i]) * inv_l, __uint_as_float(v[i + 1]) * inv_l,
                                      __uint_as_float(v[i + 2]) * inv_l, __uint_as_float(v[i + 3]) * inv_l);
          }
        }
        if (live) p.lse_part[static_cast<size_t>(seg.out_row + qrow) * p.num_q_heads + head] = lse;
      }
      tc_fence_before();
      mbar_arrive(&sm.o_empty[h]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace fwd
}  // namespace fcpb
