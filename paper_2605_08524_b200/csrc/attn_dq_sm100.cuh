// K2b: query-stationary dQ kernel on sm_100a (tcgen05 + TMEM + TMA).
//
// The KV-stationary backward (attn_bwd_sm100.cuh) would have to reduce a 32 KB
// fp32 dQ partial per 64x128 tile into global memory; on B200 those reductions
// run at ~9 B/clk/SM and bound the whole backward.  Here dQ is recomputed the
// FlashAttention-2 way instead: one CTA owns 128 query rows of one head and
// streams every KV tile of its FCP segment (local and received chunks), so dQ
// accumulates in TMEM and is written once, in bf16 -- no atomics, deterministic.
//
// Per KV tile j (128 rows, all matmuls 128x128x128 bf16 -> fp32, full-rate SS):
//   S  = Q  K_j^T        -> TMEM [0,128)
//   dP = dO V_j^T        -> TMEM [128,256)
//   softmax WGs (thread == query row): P = exp2(S*c - lse2), dS = P (dP - delta)
//        -> bf16 into TMEM (double buffered); S/dP are released as soon as they are in
//        registers, so the tensor pipe computes S/dP(j+1) while dS(j) is being formed.
//   dQ += dS K_j         (TS: A = dS in TMEM)   -> TMEM [256,384)
// TMEM: S [0,128) dP [128,256) dQ [256,384) dS0 [384,448) dS1 [448,512).
// Shared memory holds only TMA-fed operands: Q, dO, a 3-deep K ring and a 2-deep V ring
// (K(j) stays until dQ(j) has read it; the ring depth hides the ~1,300-cycle TMA latency).
// Warps: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, then four softmax/epilogue warpgroups,
// each owning 32 columns of every tile (and of dQ) for all 128 rows (a warp reaches TMEM
// lanes 32*(warp%4)..+31, so every warpgroup covers every row).  Four warps per SMSP hide
// the exp/convert dependency chains that left two warpgroups latency-bound.
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

namespace fcpb {
namespace dq {

#ifdef FCPB_TRACE
constexpr int kTraceTiles = 256;
enum DqEv { kDqKIssue, kDqKGot, kDqSdpIssue, kDqDsGot, kDqDqIssue, kDqSdpGot, kDqFreed, kDqDsArrive, kDqEvents };
__device__ unsigned long long g_trace[kDqEvents * kTraceTiles];
#define FCPB_DQTR(ev, j) do { if (blockIdx.x == 0 && (j) < kTraceTiles && (threadIdx.x & 31) == 0 && \
    ((ev) < kDqSdpGot ? true : threadIdx.x == 128)) g_trace[(ev) * kTraceTiles + (j)] = clock64(); } while (0)
#else
#define FCPB_DQTR(ev, j) do {} while (0)
#endif

constexpr int kD = 128;
constexpr int kBM = 128;                     // query rows per item
constexpr int kBN = 128;                     // kv rows per tile
constexpr int kTile = kBN * kD * 2;          // 32 KB (two SW128 panels of 64 columns)
constexpr int kPanel = kTile / 2;
constexpr int kKSlots = 3;
constexpr int kVSlots = 2;
constexpr int kSoftmaxWGs = 4;                   // each owns 128/kSoftmaxWGs columns of a tile
constexpr int kCols = kBN / kSoftmaxWGs;         // 32
constexpr int kThreads = 128 + 128 * kSoftmaxWGs;
// setmaxnreg split. setmaxnreg.inc can only take registers the CTA was given at launch
// (kThreads x kRegsLaunch, the __launch_bounds__ allocation: 65536/640 rounded down to 8),
// so the warpgroup budgets must sum to at most (1 + kSoftmaxWGs) * kRegsLaunch.
constexpr uint32_t kRegsLaunch = 96, kRegsCtl = 64, kRegsSoftmax = 104;
static_assert(kRegsCtl + kSoftmaxWGs * kRegsSoftmax <= (1 + kSoftmaxWGs) * kRegsLaunch,
              "setmaxnreg.inc would wait forever for registers that were never allocated");
constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256;
FCPB_DEV constexpr uint32_t col_ds(uint32_t b) { return 384u + 64u * b; }   // bf16 dS, 64 cols

struct Smem {
  uint8_t q[kTile];
  uint8_t dout[kTile];
  uint8_t k[kKSlots][kTile];
  uint8_t v[kVSlots][kTile];
  uint64_t qd_full, qd_empty;
  uint64_t k_full[kKSlots], k_empty[kKSlots];
  uint64_t v_full[kVSlots], v_empty[kVSlots];
  uint64_t sdp_full, sdp_free;
  uint64_t ds_full[2], ds_free[2];
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
  float scale, scale_log2;
  const float* lse2_t;     // [Hq, t_pad]  -lse*log2(e)
  const float* delta_t;    // [Hq, t_pad]  -delta
  int64_t t_pad;
  __nv_bfloat16* dq;       // [Tq, Hq, D] bf16 output
};

FCPB_DEV int item_of(int g, const Params& p) { return p.head_major ? g % p.num_items : g / p.num_q_heads; }
FCPB_DEV int head_of(int g, const Params& p) { return p.head_major ? g / p.num_items : g % p.num_q_heads; }

FCPB_DEV int kv_tiles(const FcpbKvRef& ref, int mb) {
  int n = (ref.len + kBN - 1) / kBN;
  if (ref.flags & FCPB_KV_DIAG) n = min(n, mb + 1);
  return n;
}


// 64 columns of one query row: dS = exp2(S*c + nlse) * (dP + ndelta) -> 32 bf16 pairs in TMEM
// (this row's lane, columns t_ds..t_ds+31).  kMask: column validity and causal diagonal.
template <bool kMask>
FCPB_DEV void ds_cols(const uint32_t (&s)[kCols], const uint32_t (&dp)[kCols], float c, float nlse,
                      float ndelta, uint32_t t_ds, int col0, int valid, int diag_row) {
  const float2 c2 = make_float2(c, c), nl = make_float2(nlse, nlse), nd = make_float2(ndelta, ndelta);
  uint32_t pk[kCols / 2];
#pragma unroll
  for (int u = 0; u < kCols / 2; ++u) {
    const int i = 2 * u;
    const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), c2, nl);
    float p0 = ex2(x.x), p1 = ex2(x.y);
    if (kMask) {
      const int cg = col0 + i;
      p0 = (cg < valid && cg <= diag_row) ? p0 : 0.f;
      p1 = (cg + 1 < valid && cg + 1 <= diag_row) ? p1 : 0.f;
    }
    const float2 d = __fmul2_rn(make_float2(p0, p1),
                                __fadd2_rn(make_float2(__uint_as_float(dp[i]), __uint_as_float(dp[i + 1])), nd));
    pk[u] = pack_bf16(d.x, d.y);
  }
  tmem_st16(t_ds, pk);
}

__global__ void __launch_bounds__(kThreads, 1)
attn_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
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
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_k_recv);
    tma_prefetch_desc(&tm_v_recv);
  }
  if (warp == 1 && elect_one()) {
    mbar_init(&sm.qd_full, 1);
    mbar_init(&sm.qd_empty, 1);
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVSlots; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    mbar_init(&sm.sdp_full, 1);
    mbar_init(&sm.sdp_free, 128 * kSoftmaxWGs);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.ds_full[b], 128 * kSoftmaxWGs);
      mbar_init(&sm.ds_free[b], 1);
    }
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
      // ------------------------------------------------------------ TMA producer
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t q_phase = 0, vslot = 0, v_phase = 0, kslot = 0, k_phase = 0;
        int ptile = 0;
        SchedCursor sc;
        for (int g; (g = sched_produce(sm.sched, sc, p.sched_counter)) < total;) {
          const FcpbItem it = p.items[item_of(g, p)];
          const int h = head_of(g, p);
          const int kvh = h / group;
          const FcpbSegment seg = p.segs[it.seg];
          const int row0 = seg.q_off + it.mblock * kBM;
          mbar_wait(&sm.qd_empty, q_phase ^ 1);
          q_phase ^= 1;
          mbar_arrive_expect_tx(&sm.qd_full, 2 * kTile);
          for (int half = 0; half < 2; ++half) {
            tma_load_3d(&sm.q[half * kPanel], &tm_q, &sm.qd_full, half * 64, h, row0);
            tma_load_3d(&sm.dout[half * kPanel], &tm_do, &sm.qd_full, half * 64, h, row0);
          }
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
      // ------------------------------------------------------------ MMA issuer
      const uint32_t id_kk = idesc_bf16_f32(kBM, kBN, false, false);   // S, dP
      const uint32_t id_dq = idesc_bf16_f32(kBM, kD, false, true);     // dQ += dS K (K MN-major)
      const uint32_t a_q = smem_u32(sm.q), a_do = smem_u32(sm.dout);
      const bool leader = elect_one();
      uint32_t q_phase = 0, vslot = 0, v_phase = 0, kslot = 0, k_phase = 0, sdpf_phase = 0,
               dqf_phase = 0;
      uint32_t ds_phase[2] = {0, 0}, tile = 0;
      SchedCursor sc;
      for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
        const FcpbItem it = p.items[item_of(g, p)];
        const FcpbSegment seg = p.segs[it.seg];
        int n = 0;
        for (int r = seg.kv_begin; r < seg.kv_end; ++r) n += kv_tiles(p.kvrefs[r], it.mblock);
        mbar_wait(&sm.qd_full, q_phase);
        q_phase ^= 1;
        uint32_t prev_k = 0;
        // dQ(j) += dS(j) K(j), issued once the softmax has formed dS(j)
        auto issue_dq = [&](bool first_dq, bool last) {
          const uint32_t bb = (tile - 1) & 1;
          mbar_wait(&sm.ds_full[bb], ds_phase[bb]);
          ds_phase[bb] ^= 1;
          FCPB_DQTR(kDqDsGot, (int)tile - 1);
          if (first_dq) {                     // the epilogue has drained the previous item's dQ
            mbar_wait(&sm.dq_free, dqf_phase ^ 1);
            dqf_phase ^= 1;
          }
          tc_fence_after();
          if (leader) {
            const uint32_t b_k = smem_u32(sm.k[prev_k]);
  #pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)
              mma_ts(tmem + kColDQ, tmem + col_ds(bb) + kk * 8,
                     smem_desc_sw128(b_k + kk * 2048, kPanel, 1024), id_dq, (!first_dq || kk > 0));
            mma_commit(&sm.ds_free[bb]);
            mma_commit(&sm.k_empty[prev_k]);
            if (last) mma_commit(&sm.dq_full);
          }
          __syncwarp();
          FCPB_DQTR(kDqDqIssue, (int)tile - 1);
        };
        for (int j = 0; j < n; ++j) {
          // S(j), dP(j): the softmax must hold S/dP(j-1) in registers already
          const uint32_t ks = kslot;
          mbar_wait(&sm.k_full[ks], k_phase);
          if (++kslot == kKSlots) { kslot = 0; k_phase ^= 1; }
          const uint32_t vs = vslot;
          mbar_wait(&sm.v_full[vs], v_phase);
          if (++vslot == kVSlots) { vslot = 0; v_phase ^= 1; }
          FCPB_DQTR(kDqKGot, (int)tile);
          mbar_wait(&sm.sdp_free, sdpf_phase ^ 1);
          sdpf_phase ^= 1;
          tc_fence_after();
          if (leader) {
            const uint32_t a_k = smem_u32(sm.k[ks]), a_v = smem_u32(sm.v[vs]);
  #pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
              const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
              mma_ss(tmem + kColS, smem_desc_sw128(a_q + off, 16, 1024),
                     smem_desc_sw128(a_k + off, 16, 1024), id_kk, kk > 0);
            }
  #pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
              const uint32_t off = (kk >> 2) * kPanel + (kk & 3) * 32;
              mma_ss(tmem + kColDP, smem_desc_sw128(a_do + off, 16, 1024),
                     smem_desc_sw128(a_v + off, 16, 1024), id_kk, kk > 0);
            }
            mma_commit(&sm.sdp_full);
            mma_commit(&sm.v_empty[vs]);
            if (j == n - 1) mma_commit(&sm.qd_empty);   // Q / dO no longer read by this item
          }
          __syncwarp();
          FCPB_DQTR(kDqSdpIssue, (int)tile);
          if (j > 0) issue_dq(j == 1, false);           // dQ(j-1) overlaps softmax(j)
          prev_k = ks;
          ++tile;
        }
        issue_dq(n == 1, true);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    reg_alloc<kRegsSoftmax>();
    const int part = (warp - 4) >> 2;                      // which 32-column slice of the tile
    const int row = (warp & 3) * 32 + lane_id();
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_bits + kColS + part * kCols;
    const uint32_t t_dp = tmem + lane_bits + kColDP + part * kCols;
    const uint32_t t_ds0 = tmem + lane_bits + col_ds(0) + part * (kCols / 2);
    uint32_t sdp_phase = 0, dq_phase = 0, tile = 0;
    uint32_t dsf_phase[2] = {0, 0};
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
      for (int r = seg.kv_begin; r < seg.kv_end; ++r) {
        const FcpbKvRef ref = p.kvrefs[r];
        const int nt = kv_tiles(ref, it.mblock);
        const bool diag = ref.flags & FCPB_KV_DIAG;
        for (int t = 0; t < nt; ++t, ++tile) {
          const uint32_t b = tile & 1;
          const int valid = live ? ref.len - t * kBN : 0;    // dead rows contribute nothing
          const bool on_diag = diag && t == it.mblock;
          // tcgen05.st inside ds_cols is .sync.aligned: the path must be warp-uniform
          const bool plain = __all_sync(0xffffffffu, valid >= kBN && !on_diag);
          const int diag_row = on_diag ? row : kBN;           // col <= row on the diagonal tile
          mbar_wait(&sm.sdp_full, sdp_phase);
          sdp_phase ^= 1;
          FCPB_DQTR(kDqSdpGot, (int)tile);
          tc_fence_after();
          uint32_t sv[kCols], dv[kCols];
          tmem_ld32(t_s, sv);
          tmem_ld32(t_dp, dv);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&sm.sdp_free);                          // S/dP(j) in registers
          FCPB_DQTR(kDqFreed, (int)tile);
          mbar_wait(&sm.ds_free[b], dsf_phase[b] ^ 1);        // dQ(j-2) has read buffer b
          dsf_phase[b] ^= 1;
          const uint32_t t_ds = t_ds0 + b * 64;
          if (plain)
            ds_cols<false>(sv, dv, p.scale_log2, nlse, ndel, t_ds, part * kCols, kBN, kBN);
          else
            ds_cols<true>(sv, dv, p.scale_log2, nlse, ndel, t_ds, part * kCols, valid, diag_row);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&sm.ds_full[b]);
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
