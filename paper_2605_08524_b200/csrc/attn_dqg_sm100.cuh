// K2c: dQ from materialised dS tiles -- a grouped GEMM on sm_100a (tcgen05 + TMEM + TMA).
//
// When the rank's dS tiles fit in HBM, the dK/dV kernel (attn_bwd_sm100.cuh) writes every
// bf16 dS^T tile it forms (128 kv x 128 q, one per (KV block, Q block, q head)), and dQ
// needs no recomputation of S, dP or the softmax:
//     dQ[q tile, h] = scale * sum over its KV tiles  dS[q, kv] K[kv, :]
// A = dS, read from the dS^T tile stored [q/8][kv][8 q] -- the no-swizzle MN-major canonical
// layout, fetched with one 1-D bulk copy -- and B = K ([kv][d], d contiguous: SW128 MN-major).  One CTA per SM, one item = (Q block of a segment, q head), a
// 3-deep ring of (dS^T, K) tile pairs fed by TMA, dQ accumulated in TMEM (double-buffered
// across items so the next item's MMAs overlap the epilogue), a bf16 epilogue.  The
// recompute kernel (attn_dq_sm100.cuh) stays the path for batches whose dS does not fit
// (C3: 2.5 TB).
// Warps: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 epilogue (thread == query row).
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

namespace fcpb {
namespace dqg {

constexpr int kD = 128;
constexpr int kBM = 128;                     // query rows per item
constexpr int kBN = 128;                     // kv rows per tile
constexpr int kTile = kBN * kD * 2;          // 32 KB (two SW128 panels of 64 columns)
constexpr int kPanel = kTile / 2;
constexpr int kStages = 3;
constexpr int kThreads = 256;

struct Smem {
  uint8_t ds[kStages][kTile];
  uint8_t k[kStages][kTile];
  uint64_t full[kStages], empty[kStages];
  uint64_t dq_full[2], dq_free[2];
  SchedRing sched;
  uint32_t tmem_base;
};

struct Params {
  int* sched_counter;
  const FcpbSegment* segs;
  const FcpbKvRef* kvrefs;
  const FcpbItem* items;
  const __nv_bfloat16* ds;   // dS^T tiles [tiles][16][128][8]
  const int32_t* pair_ids;   // per (item, kv tile), item-major (worklist.build_ds_tiles)
  const int32_t* pair_off;   // per item: first entry in pair_ids
  int32_t num_items;
  int32_t num_q_heads, num_kv_heads;
  int32_t head_major, hm_lead;
  float scale;
  __nv_bfloat16* dq;         // [Tq, Hq, D]
  int32_t stack_tails;       // as fcpb_attn_bwd: a Q block with <= 64 rows has one dS^T tile
                             // for q-heads (h, h+1), h even, rows stacked 0-63 / 64-127
};

constexpr int kStackRows = 64;
// Item (Q block, head h) of a stacked tail: the even head computes both heads' rows; the odd
// head's item is empty.
FCPB_DEV bool stacked(const Params& p, const FcpbSegment& seg, const FcpbItem& it) {
  return p.stack_tails && seg.q_len - it.mblock * kBM <= kStackRows;
}

FCPB_DEV int kv_tiles(const FcpbKvRef& ref, int mb) {
  int n = (ref.len + kBN - 1) / kBN;
  if (ref.flags & FCPB_KV_DIAG) n = min(n, mb + 1);
  return n;
}

__global__ void __launch_bounds__(kThreads, 1)
attn_dqg_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_k_recv,
                const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id();
  const int H = p.num_q_heads;
  const int group = H / p.num_kv_heads;
  const int total = p.num_items * H;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_k_recv);
  }
  if (warp == 1 && elect_one()) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.dq_full[b], 1);
      mbar_init(&sm.dq_free[b], 128);
    }
    sched_init(sm.sched, 1 + 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<256>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();     // K tiles: reused by other Q blocks
      const uint64_t once = policy_evict_first();    // dS tiles: read exactly once
      uint32_t slot = 0, phase = 0;
      SchedCursor sc;
      for (int g; (g = sched_produce(sm.sched, sc, p.sched_counter)) < total;) {
        int item, h;
        grid_map(g, p.num_items, H, p.head_major, p.hm_lead, item, h);
        const FcpbItem it = p.items[item];
        const FcpbSegment seg = p.segs[it.seg];
        if (stacked(p, seg, it) && (h & 1)) continue;
        const int kvh = h / group;
        int j = p.pair_off[item];
        for (int r = seg.kv_begin; r < seg.kv_end; ++r) {
          const FcpbKvRef ref = p.kvrefs[r];
          const bool recv = ref.flags & FCPB_KV_RECV;
          const int nt = kv_tiles(ref, it.mblock);
          for (int t = 0; t < nt; ++t, ++j) {
            mbar_wait(&sm.empty[slot], phase ^ 1);
            mbar_arrive_expect_tx(&sm.full[slot], 2 * kTile);
            const size_t tile = static_cast<size_t>(p.pair_ids[j]) * H + h;
            bulk_load_hint(sm.ds[slot], p.ds + tile * (kBN * kBM), kTile, &sm.full[slot], once);
            for (int half = 0; half < 2; ++half)
              tma_load_3d_hint(&sm.k[slot][half * kPanel], recv ? &tm_k_recv : &tm_k, &sm.full[slot],
                               half * 64, kvh, ref.off + t * kBN, keep);
            if (++slot == kStages) { slot = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t id = idesc_bf16_f32(kBM, kD, true, true);   // A (dS) and B (K) MN-major
    const bool leader = elect_one();
    uint32_t slot = 0, phase = 0, item_par = 0;
    uint32_t free_phase[2] = {0, 0};
    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      int item, h;
      grid_map(g, p.num_items, H, p.head_major, p.hm_lead, item, h);
      const FcpbItem it = p.items[item];
      const FcpbSegment seg = p.segs[it.seg];
      if (stacked(p, seg, it) && (h & 1)) continue;
      int n = 0;
      for (int r = seg.kv_begin; r < seg.kv_end; ++r) n += kv_tiles(p.kvrefs[r], it.mblock);
      const uint32_t b = item_par;
      mbar_wait(&sm.dq_free[b], free_phase[b] ^ 1);         // epilogue drained this buffer
      free_phase[b] ^= 1;
      tc_fence_after();
      const uint32_t d_col = tmem + b * kD;
      for (int j = 0; j < n; ++j) {
        mbar_wait(&sm.full[slot], phase);
        tc_fence_after();
        if (leader) {
          const uint32_t a = smem_u32(sm.ds[slot]), bk = smem_u32(sm.k[slot]);
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk)
            mma_ss(d_col, smem_desc_noswz(a + kk * 256, 128, kBN * 16),
                   smem_desc_sw128(bk + kk * 2048, kPanel, 1024), id, (j > 0 || kk > 0));
          mma_commit(&sm.empty[slot]);
          if (j == n - 1) mma_commit(&sm.dq_full[b]);
        }
        __syncwarp();
        if (++slot == kStages) { slot = 0; phase ^= 1; }
      }
      item_par ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (thread == q row)
    const int row = (warp & 3) * 32 + lane_id();
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t item_par = 0;
    uint32_t full_phase[2] = {0, 0};
    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      int item, h;
      grid_map(g, p.num_items, H, p.head_major, p.hm_lead, item, h);
      const FcpbItem it = p.items[item];
      const FcpbSegment seg = p.segs[it.seg];
      const bool stk = stacked(p, seg, it);
      if (stk && (h & 1)) continue;
      const uint32_t b = item_par;
      item_par ^= 1;
      mbar_wait(&sm.dq_full[b], full_phase[b]);
      full_phase[b] ^= 1;
      tc_fence_after();
      // stacked: accumulator rows 64-127 are head h+1's rows 0-63
      const int qpos = it.mblock * kBM + (stk ? (row & (kStackRows - 1)) : row);
      const int hh = stk ? h + (row >> 6) : h;
      const bool live = qpos < seg.q_len;
      __nv_bfloat16* dst = p.dq + (static_cast<size_t>(seg.q_off + (live ? qpos : 0)) * H + hh) * kD;
#pragma unroll
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_bits + b * kD + c * 32, v);
        tmem_wait_ld();
        if (live) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
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
      mbar_arrive(&sm.dq_free[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

}  // namespace dqg
}  // namespace fcpb
