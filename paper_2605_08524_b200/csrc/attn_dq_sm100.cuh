// K2b: query-stationary dQ kernel on sm_100a (tcgen05 + TMEM + TMA).
//
// The KV-stationary backward (attn_bwd_sm100.cuh) would have to reduce a fp32 dQ
// partial per tile into global memory; on B200 those reductions run at ~9 B/clk/SM
// and bound the whole backward.  Here dQ is recomputed the FlashAttention-2 way
// instead: one CTA owns 128 query rows of one head and streams every KV tile of its
// FCP segment (local and received chunks), so dQ accumulates in TMEM and is written
// once, in bf16 -- no atomics, deterministic.
//
// Q and dO are item-stationary, so they live in TMEM (bf16, 64 columns each) and the
// two score matmuls are TS MMAs that read only K/V from shared memory.  (As SS MMAs at
// N=128 they sat exactly on the 128 B/clk shared-memory operand limit and ran ~1.7x
// slow once the TMA writes of the K/V stream competed for the same port.)
// Per KV tile j (128 rows, all matmuls 128x128x128 bf16 -> fp32):
//   S  = Q  K_j^T    (TS: A = Q  in TMEM)  -> TMEM S  [0,128)
//   dP = dO V_j^T    (TS: A = dO in TMEM)  -> TMEM dP [128,256)
//   softmax WGs (thread == query row, warpgroup w owns kv columns [32w, 32w+32)):
//     phase A: P = exp2(S*c - lse2) in registers (S is released right after the load)
//     phase B: dS = P (dP - delta) -> bf16, in place over the first 16 of its dP columns
//   dQ += dS K_j     (TS: A = dS in TMEM)  -> TMEM dQ [256,384)
// TMEM: S [0,128) dP/dS [128,256) dQ [256,384) Q [384,448) dO [448,512).
// Issue order S(j+1), dQ(j), dP(j+1): the in-order pipe keeps dP(j+1) from overwriting
// dS(j) before dQ(j) read it, and phase A of tile j+1 overlaps dQ(j)/dP(j+1).
// Shared memory holds only the K ring (K(j) stays until dQ(j) read it) and the V ring.
// Warps: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, then four softmax/epilogue warpgroups
// (a warp reaches TMEM lanes 32*(warp%4)..+31, so every warpgroup covers every row).
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

#ifndef FCPB_DQ_POLY
#define FCPB_DQ_POLY 1    // polynomial exp2 pairs per 4 (0..3)
#endif
#ifndef FCPB_DQ_SPIN
#define FCPB_DQ_SPIN 1    // 1: MMA warp spins on ds_full; 2: also the softmax's dP wait
#endif

namespace fcpb {
namespace dq {

#ifdef FCPB_TRACE
constexpr int kTraceTiles = 256;
enum DqEv { kDqKIssue, kDqKGot, kDqSIssue, kDqDsGot, kDqDqIssue, kDqSGot, kDqFreed, kDqDpGot,
            kDqDsArrive, kDqEvents };
__device__ unsigned long long g_trace[kDqEvents * kTraceTiles];
#define FCPB_DQTR(ev, j) do { if (blockIdx.x == 0 && (j) < kTraceTiles && (threadIdx.x & 31) == 0 && \
    ((ev) < kDqSGot ? true : threadIdx.x == 128)) g_trace[(ev) * kTraceTiles + (j)] = clock64(); } while (0)
#else
#define FCPB_DQTR(ev, j) do {} while (0)
#endif

constexpr int kD = 128;
constexpr int kBM = 128;                     // query rows per item
constexpr int kBN = 128;                     // kv rows per tile
constexpr int kTile = kBN * kD * 2;          // 32 KB (two SW128 panels of 64 columns)
constexpr int kPanel = kTile / 2;
constexpr int kKSlots = 4;
constexpr int kVSlots = 3;
constexpr int kSoftmaxWGs = 4;                   // each owns 128/kSoftmaxWGs columns of a tile
constexpr int kCols = kBN / kSoftmaxWGs;         // 32
constexpr int kThreads = 128 + 128 * kSoftmaxWGs;
// setmaxnreg split. setmaxnreg.inc can only take registers the CTA was given at launch
// (kThreads x kRegsLaunch, the __launch_bounds__ allocation: 65536/640 rounded down to 8),
// so the warpgroup budgets must sum to at most (1 + kSoftmaxWGs) * kRegsLaunch.
constexpr uint32_t kRegsLaunch = 96, kRegsCtl = 64, kRegsSoftmax = 104;
static_assert(kRegsCtl + kSoftmaxWGs * kRegsSoftmax <= (1 + kSoftmaxWGs) * kRegsLaunch,
              "setmaxnreg.inc would wait forever for registers that were never allocated");
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColQ = 384, kColDO = 448;

// TMEM column of the bf16 dS chunk kk (16 kv columns = 8 TMEM columns): warpgroup w keeps
// its 32 columns in the first 16 TMEM columns of its own dP slice.
FCPB_DEV constexpr uint32_t ds_col(int kk) {
  return kColDP + static_cast<uint32_t>((kk >> 1) * kCols + (kk & 1) * 8);
}

struct Smem {
  uint8_t k[kKSlots][kTile];
  uint8_t v[kVSlots][kTile];
  uint64_t k_full[kKSlots], k_empty[kKSlots];
  uint64_t v_full[kVSlots], v_empty[kVSlots];
  uint64_t qd_full;                  // Q / dO of the item are in TMEM
  uint64_t s_full, s_free, dp_full, ds_full;
  uint64_t dq_full, dq_free;
  SchedRing sched;
  uint32_t tmem_base;
};

struct Params {
  int* sched_counter;      // dynamic tile scheduler (zeroed before launch)
  const FcpbSegment* segs;
  const FcpbKvRef* kvrefs;
  const FcpbItem* items;
  int32_t num_items;
  int32_t num_q_heads, num_kv_heads;
  int32_t head_major;      // grid index -> (item, head) mapping, see item_of()
  int32_t hm_lead;         // head_major: items run heads-adjacent before the head-major rest
  float scale, scale_log2;
  const __nv_bfloat16* q;  // [Tq, Hq, D]
  const __nv_bfloat16* dout;
  const float* lse2_t;     // [Hq, t_pad]  -lse*log2(e)
  const float* delta_t;    // [Hq, t_pad]  -delta
  int64_t t_pad;
  __nv_bfloat16* dq;       // [Tq, Hq, D] bf16 output
};

FCPB_DEV int item_of(int g, const Params& p) {
  int it, h;
  grid_map(g, p.num_items, p.num_q_heads, p.head_major, p.hm_lead, it, h);
  return it;
}
FCPB_DEV int head_of(int g, const Params& p) {
  int it, h;
  grid_map(g, p.num_items, p.num_q_heads, p.head_major, p.hm_lead, it, h);
  return h;
}

FCPB_DEV int kv_tiles(const FcpbKvRef& ref, int mb) {
  int n = (ref.len + kBN - 1) / kBN;
  if (ref.flags & FCPB_KV_DIAG) n = min(n, mb + 1);
  return n;
}

// Phase A, 32 kv columns of one query row: P = exp2(S*c + nlse).  kMask: column validity
// and the causal diagonal.  A quarter of the pairs go to the FMA pipe (FA4-style): the
// MUFU pipe alone needs 4 warps x 32 ex2 x 8 cycles per SMSP per tile.
template <bool kMask>
FCPB_DEV void p_cols(const uint32_t (&s)[kCols], float c, float nlse, float (&pr)[kCols],
                     int col0, int valid, int diag_row) {
  const float2 c2 = make_float2(c, c), nl = make_float2(nlse, nlse);
#pragma unroll
  for (int u = 0; u < kCols / 2; ++u) {
    const int i = 2 * u;
    const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), c2, nl);
    float p0, p1;
    const bool use_poly = FCPB_DQ_POLY == 0 ? false : FCPB_DQ_POLY == 1 ? (u & 3) == 3
                          : FCPB_DQ_POLY == 2 ? (u & 1) != 0 : (u & 3) != 0;
    if (use_poly) {
      const float2 e = ex2_poly2(x);
      p0 = e.x;
      p1 = e.y;
    } else {
      p0 = ex2(x.x);
      p1 = ex2(x.y);
    }
    if (kMask) {
      const int cg = col0 + i;
      p0 = (cg < valid && cg <= diag_row) ? p0 : 0.f;
      p1 = (cg + 1 < valid && cg + 1 <= diag_row) ? p1 : 0.f;
    }
    pr[i] = p0;
    pr[i + 1] = p1;
  }
}

// Phase B: dS = P (dP + ndelta) -> 16 bf16 pairs at t_ds.
FCPB_DEV void ds_cols(const float (&pr)[kCols], const uint32_t (&dp)[kCols], float ndelta,
                      uint32_t t_ds) {
  const float2 nd = make_float2(ndelta, ndelta);
  uint32_t pk[kCols / 2];
#pragma unroll
  for (int u = 0; u < kCols / 2; ++u) {
    const int i = 2 * u;
    const float2 d = __fmul2_rn(make_float2(pr[i], pr[i + 1]),
                                __fadd2_rn(make_float2(__uint_as_float(dp[i]), __uint_as_float(dp[i + 1])), nd));
    pk[u] = pack_bf16(d.x, d.y);
  }
  tmem_st16(t_ds, pk);
}

__global__ void __launch_bounds__(kThreads, 1)
attn_dq_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
               const __grid_constant__ CUtensorMap tm_k_recv,
               const __grid_constant__ CUtensorMap tm_v_recv, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id();
  const int H = p.num_q_heads;
  const int group = H / p.num_kv_heads;
  const int total = p.num_items * H;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_k_recv);
    tma_prefetch_desc(&tm_v_recv);
  }
  if (warp == 1 && elect_one()) {
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVSlots; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    mbar_init(&sm.qd_full, 128 * kSoftmaxWGs);
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.s_free, 128 * kSoftmaxWGs);
    mbar_init(&sm.dp_full, 1);
    mbar_init(&sm.ds_full, 128 * kSoftmaxWGs);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_free, 128 * kSoftmaxWGs);
    sched_init(sm.sched, 1 + 4 * kSoftmaxWGs);
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
      // ---------------------------------------------------------- TMA producer (K/V stream)
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t vslot = 0, v_phase = 0, kslot = 0, k_phase = 0;
        int ptile = 0;
        SchedCursor sc;
        for (int g; (g = sched_produce(sm.sched, sc, p.sched_counter)) < total;) {
          const FcpbItem it = p.items[item_of(g, p)];
          const int kvh = head_of(g, p) / group;
          const FcpbSegment seg = p.segs[it.seg];
          for (int r = seg.kv_begin; r < seg.kv_end; ++r) {
            const FcpbKvRef ref = p.kvrefs[r];
            const bool recv = ref.flags & FCPB_KV_RECV;
            const int nt = kv_tiles(ref, it.mblock);
            for (int t = 0; t < nt; ++t) {
              const int krow = ref.off + t * kBN;
              mbar_wait(&sm.k_empty[kslot], k_phase ^ 1);
              mbar_arrive_expect_tx(&sm.k_full[kslot], kTile);
              for (int half = 0; half < 2; ++half)
                tma_load_3d_hint(&sm.k[kslot][half * kPanel], recv ? &tm_k_recv : &tm_k,
                                 &sm.k_full[kslot], half * 64, kvh, krow, keep);
              if (++kslot == kKSlots) { kslot = 0; k_phase ^= 1; }
              mbar_wait(&sm.v_empty[vslot], v_phase ^ 1);
              mbar_arrive_expect_tx(&sm.v_full[vslot], kTile);
              for (int half = 0; half < 2; ++half)
                tma_load_3d_hint(&sm.v[vslot][half * kPanel], recv ? &tm_v_recv : &tm_v,
                                 &sm.v_full[vslot], half * 64, kvh, krow, keep);
              if (++vslot == kVSlots) { vslot = 0; v_phase ^= 1; }
              FCPB_DQTR(kDqKIssue, ptile); ++ptile;
            }
          }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      const uint32_t id_kk = idesc_bf16_f32(kBM, kBN, false, false);   // S, dP
      const uint32_t id_dq = idesc_bf16_f32(kBM, kD, false, true);     // dQ += dS K (K MN-major)
      const bool leader = elect_one();
      uint32_t qd_phase = 0, vslot = 0, v_phase = 0, kslot = 0, k_phase = 0, sf_phase = 0,
               ds_phase = 0, dqf_phase = 0;
      uint32_t tile = 0;
      // S = Q K^T / dP = dO V^T: A (Q or dO, bf16 [128 x 128]) from TMEM, B from the ring.
      auto issue_score = [&](uint32_t a_col, uint32_t b_base, uint32_t d_col, uint64_t* done,
                             uint64_t* release) {
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
            mma_ts(tmem + d_col, tmem + a_col + kk * 8, smem_desc_sw128(b_base + off, 16, 1024),
                   id_kk, kk > 0);
          }
          mma_commit(done);
          if (release) mma_commit(release);
        }
        __syncwarp();
      };
      SchedCursor sc;
      for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
        const FcpbItem it = p.items[item_of(g, p)];
        const FcpbSegment seg = p.segs[it.seg];
        int n = 0;
        for (int r = seg.kv_begin; r < seg.kv_end; ++r) n += kv_tiles(p.kvrefs[r], it.mblock);
        mbar_wait(&sm.qd_full, qd_phase);              // Q / dO of this item are in TMEM
        qd_phase ^= 1;
        tc_fence_after();
        // prologue: S(0), dP(0).  Every tile's S is released once (s_free); the previous
        // item's last release is consumed here.
        uint32_t ks = kslot;
        mbar_wait(&sm.k_full[ks], k_phase);
        if (++kslot == kKSlots) { kslot = 0; k_phase ^= 1; }
        FCPB_DQTR(kDqKGot, (int)tile);
        if (tile > 0) {
          mbar_wait(&sm.s_free, sf_phase);
          sf_phase ^= 1;
        }
        tc_fence_after();
        issue_score(kColQ, smem_u32(sm.k[ks]), kColS, &sm.s_full, nullptr);
        FCPB_DQTR(kDqSIssue, (int)tile);
        {
          const uint32_t vs = vslot;
          mbar_wait(&sm.v_full[vs], v_phase);
          if (++vslot == kVSlots) { vslot = 0; v_phase ^= 1; }
          tc_fence_after();
          issue_score(kColDO, smem_u32(sm.v[vs]), kColDP, &sm.dp_full, &sm.v_empty[vs]);
        }
        for (int j = 0; j < n; ++j, ++tile) {
          const uint32_t ks_j = ks;
          if (j + 1 < n) {
            ks = kslot;
            mbar_wait(&sm.k_full[ks], k_phase);
            if (++kslot == kKSlots) { kslot = 0; k_phase ^= 1; }
            FCPB_DQTR(kDqKGot, (int)tile + 1);
            mbar_wait(&sm.s_free, sf_phase);             // softmax holds S(j) in registers
            sf_phase ^= 1;
            tc_fence_after();
            issue_score(kColQ, smem_u32(sm.k[ks]), kColS, &sm.s_full, nullptr);
            FCPB_DQTR(kDqSIssue, (int)tile + 1);
          }
          if (FCPB_DQ_SPIN >= 1) mbar_wait_spin(&sm.ds_full, ds_phase);
          else mbar_wait(&sm.ds_full, ds_phase);
          ds_phase ^= 1;
          FCPB_DQTR(kDqDsGot, (int)tile);
          if (j == 0) {                                   // epilogue drained the previous dQ
            mbar_wait(&sm.dq_free, dqf_phase ^ 1);
            dqf_phase ^= 1;
          }
          tc_fence_after();
          if (leader) {
            const uint32_t b_k = smem_u32(sm.k[ks_j]);
#pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)
              mma_ts(tmem + kColDQ, tmem + ds_col(kk),
                     smem_desc_sw128(b_k + kk * 2048, kPanel, 1024), id_dq, (j > 0 || kk > 0));
            mma_commit(&sm.k_empty[ks_j]);
            if (j == n - 1) mma_commit(&sm.dq_full);
          }
          __syncwarp();
          FCPB_DQTR(kDqDqIssue, (int)tile);
          if (j + 1 < n) {
            const uint32_t vs = vslot;
            mbar_wait(&sm.v_full[vs], v_phase);
            if (++vslot == kVSlots) { vslot = 0; v_phase ^= 1; }
            tc_fence_after();
            issue_score(kColDO, smem_u32(sm.v[vs]), kColDP, &sm.dp_full, &sm.v_empty[vs]);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    reg_alloc<kRegsSoftmax>();
    const int part = (warp - 4) >> 2;                      // kv columns [32 part, +32) of a tile
    const int row = (warp & 3) * 32 + lane_id();
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_bits + kColS + part * kCols;
    const uint32_t t_dp = tmem + lane_bits + kColDP + part * kCols;
    uint32_t s_phase = 0, dp_phase = 0, dq_phase = 0, tile = 0;
    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      const FcpbItem it = p.items[item_of(g, p)];
      const int h = head_of(g, p);
      const FcpbSegment seg = p.segs[it.seg];
      const int qpos = it.mblock * kBM + row;                // row inside the Q chunk
      const bool live = qpos < seg.q_len;
      const int64_t tl = static_cast<int64_t>(h) * p.t_pad + seg.q_off + (live ? qpos : 0);
      const float nlse = live ? p.lse2_t[tl] : 0.f;
      const float ndel = live ? p.delta_t[tl] : 0.f;
      // ---- Q / dO of this row, d columns [32 part, +32), into TMEM as bf16 pairs.  The
      // previous item's S/dP completed before its dQ(last), which this warpgroup waited
      // for in its epilogue, so the columns are free.
      {
        const size_t off = (static_cast<size_t>(seg.q_off + (live ? qpos : 0)) * H + h) * kD + part * 32;
        const uint4* qs = reinterpret_cast<const uint4*>(p.q + off);
        const uint4* ds = reinterpret_cast<const uint4*>(p.dout + off);
        uint32_t qv[16], dv[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 a = live ? __ldg(qs + i) : make_uint4(0, 0, 0, 0);
          const uint4 b = live ? __ldg(ds + i) : make_uint4(0, 0, 0, 0);
          qv[4 * i] = a.x; qv[4 * i + 1] = a.y; qv[4 * i + 2] = a.z; qv[4 * i + 3] = a.w;
          dv[4 * i] = b.x; dv[4 * i + 1] = b.y; dv[4 * i + 2] = b.z; dv[4 * i + 3] = b.w;
        }
        tmem_st16(tmem + lane_bits + kColQ + part * 16, qv);
        tmem_st16(tmem + lane_bits + kColDO + part * 16, dv);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&sm.qd_full);
      }
      for (int r = seg.kv_begin; r < seg.kv_end; ++r) {
        const FcpbKvRef ref = p.kvrefs[r];
        const int nt = kv_tiles(ref, it.mblock);
        const bool diag = ref.flags & FCPB_KV_DIAG;
        for (int t = 0; t < nt; ++t, ++tile) {
          const int valid = live ? ref.len - t * kBN : 0;    // dead rows contribute nothing
          const bool on_diag = diag && t == it.mblock;
          const bool plain = valid >= kBN && !on_diag;
          const int diag_row = on_diag ? row : kBN;           // col <= row on the diagonal tile
          float pr[kCols];
          mbar_wait(&sm.s_full, s_phase);
          s_phase ^= 1;
          FCPB_DQTR(kDqSGot, (int)tile);
          tc_fence_after();
          {
            uint32_t sv[kCols];
            tmem_ld32(t_s, sv);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&sm.s_free);                          // S(j) in registers
            FCPB_DQTR(kDqFreed, (int)tile);
            if (plain)
              p_cols<false>(sv, p.scale_log2, nlse, pr, 0, kBN, kBN);
            else
              p_cols<true>(sv, p.scale_log2, nlse, pr, part * kCols, valid, diag_row);
          }
          if (FCPB_DQ_SPIN >= 2) mbar_wait_spin(&sm.dp_full, dp_phase);
          else mbar_wait(&sm.dp_full, dp_phase);
          dp_phase ^= 1;
          FCPB_DQTR(kDqDpGot, (int)tile);
          tc_fence_after();
          {
            uint32_t dv[kCols];
            tmem_ld32(t_dp, dv);
            tmem_wait_ld();
            ds_cols(pr, dv, ndel, t_dp);                      // in place over dP's first 16 cols
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&sm.ds_full);
          FCPB_DQTR(kDqDsArrive, (int)tile);
        }
      }
      // ---- epilogue: this warpgroup's 32 columns of dQ * scale -> bf16
      mbar_wait(&sm.dq_full, dq_phase);
      dq_phase ^= 1;
      tc_fence_after();
      {
        uint32_t v[32];
        tmem_ld32(tmem + lane_bits + kColDQ + part * kCols, v);
        tmem_wait_ld();
        if (live) {
          __nv_bfloat16* dst = p.dq + (static_cast<size_t>(seg.q_off + qpos) * H + h) * kD + part * kCols;
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(v[i + 0]) * p.scale, __uint_as_float(v[i + 1]) * p.scale);
            w.y = pack_bf16(__uint_as_float(v[i + 2]) * p.scale, __uint_as_float(v[i + 3]) * p.scale);
            w.z = pack_bf16(__uint_as_float(v[i + 4]) * p.scale, __uint_as_float(v[i + 5]) * p.scale);
            w.w = pack_bf16(__uint_as_float(v[i + 6]) * p.scale, __uint_as_float(v[i + 7]) * p.scale);
            d4[i / 8] = w;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.dq_free);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace dq
}  // namespace fcpb
