// K2: varlen block-pair attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// Work item = one 128-row KV block of one KV chunk (local or received) for one KV
// head.  The CTA streams every (Q chunk, 64-row Q block, q-head of the GQA group)
// that attends to it; dK/dV accumulate in TMEM and are written once (no atomics).
// dQ is produced by the query-stationary kernel in attn_dq_sm100.cuh: reducing a
// 32 KB fp32 dQ partial per tile from here measured ~3,750 cycles per tile on B200
// (~9 B/clk/SM of reduction throughput, TMA reduce-add and red.global alike), 2.3x
// the tile's tensor time.
//
// Per Q tile j (64 query rows):
//   S^T  = K  Q_j^T   M128 N64  K128 (SS)  -> TMEM S        (fp32)
//   dP^T = V  dO_j^T  M128 N64  K128 (SS)  -> TMEM dP
//   softmax WG (thread == kv row): loads S^T, dP^T rows, frees TMEM at once, then
//        P^T = exp2(S^T*c - lse2[q]),  dS^T = P^T (dP^T - delta[q])   -> bf16 smem
//        (SW128 rows of 64 q, double buffered)
//   dV  += P^T  dO_j  M128 N128 K64  (SS)  -> TMEM dV
//   dK  += dS^T Q_j   M128 N128 K64  (SS)  -> TMEM dK
// TMEM (512 cols): dV [0,128) dK [128,256) S [256,320) dP [320,384)
//                  P0 [384,416) dS0 [416,448) P1 [448,480) dS1 [480,512)
// The tensor pipe computes S/dP of tile j+1 while the softmax of tile j runs.
// Warps: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 softmax, w8-11 dK/dV epilogue.
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

namespace fcpb {
namespace bwd {

#ifdef FCPB_TRACE
// Debug timeline of CTA 0: [event][tile] clock64 stamps (see scripts/trace_bwd.py).
constexpr int kTraceTiles = 256;
enum TraceEv { kTrQdIssue, kTrQdGot, kTrSdpIssue, kTrPdsGot, kTrAccIssue, kTrSdpGot, kTrLoaded,
               kTrPfreeGot, kTrPdsArrive, kTrDqGot, kTrDqDone, kTrEvents };
__device__ unsigned long long g_trace[kTrEvents * kTraceTiles];
#define FCPB_TR(ev, j) do { if (blockIdx.x == 0 && (j) < kTraceTiles && (threadIdx.x & 31) == 0 && \
    ((ev) < kTrSdpGot || (ev) >= kTrDqGot ? true : threadIdx.x == 128)) \
    g_trace[(ev) * kTraceTiles + (j)] = clock64(); } while (0)
#else
#define FCPB_TR(ev, j) do {} while (0)
#endif

constexpr int kD = 128;
constexpr int kBK = 128;                        // kv rows per item
constexpr int kBQ = 64;                         // q rows per tile
constexpr int kKVBytes = kBK * kD * 2;          // 32 KB (two 16 KB SW128 panels)
constexpr int kKVPanel = kKVBytes / 2;
constexpr int kQBytes = kBQ * kD * 2;           // 16 KB (two 8 KB panels)
constexpr int kQPanel = kQBytes / 2;
constexpr int kPBytes = kBK * kBQ * 2;          // 16 KB: 128 kv rows x 64 q (one SW128 panel)
constexpr int kStages = 4;
constexpr int kThreads = 384;
constexpr uint32_t kColDV = 0, kColDK = 128, kColS = 256, kColDP = 320;
// bf16 P^T / dS^T, 32 columns each, double buffered: P_b = 384 + 64b, dS_b = 416 + 64b
FCPB_DEV constexpr uint32_t col_p(uint32_t b) { return 384u + 64u * b; }
FCPB_DEV constexpr uint32_t col_ds(uint32_t b) { return 416u + 64u * b; }

struct KvSeg { int32_t kv_off, kv_len, flags, q_begin, q_end, pad_; };
struct QRef { int32_t q_off, q_len, diag, pad_; };
struct Item { int32_t kvseg, nblock; };

struct Smem {
  uint8_t k[kKVBytes];
  uint8_t v[kKVBytes];
  uint8_t q[kStages][kQBytes];
  uint8_t dout[kStages][kQBytes];
  float lse2[kStages][kBQ];         // lse * log2(e), per q column
  float delta[kStages][kBQ];
  uint64_t kv_full, kv_empty;
  uint64_t qd_full[kStages], qd_empty[kStages];
  uint64_t sdp_full, sdp_free;
  uint64_t pds_full[2], pds_free[2];
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
  float scale;            // softmax scale
  float scale_log2;       // scale * log2(e)
  const float* lse2_t;    // [Hq, t_pad] lse * log2(e)
  const float* delta_t;   // [Hq, t_pad]
  int64_t t_pad;
  int32_t q_tokens;
  float* dk;              // local  [Tkv, Hkv, D] fp32
  float* dv;
  float* dk_recv;         // recv   [Tr, Hkv, D] fp32
  float* dv_recv;
};

// Grid index -> (item, kv head).  head_major: neighbouring CTAs run neighbouring items of
// one head (they stream the same Q/dO tiles -> L2 reuse); else the heads of one item.
FCPB_DEV int item_of(int g, const Params& p) { return p.head_major ? g % p.num_items : g / p.num_kv_heads; }
FCPB_DEV int head_of(int g, const Params& p) { return p.head_major ? g / p.num_items : g % p.num_kv_heads; }

// Q blocks (64 rows) of `qr` that see KV block `nb` (128 rows): diagonal -> mb >= 2nb.
FCPB_DEV int q_first_block(const QRef& qr, int nb) { return qr.diag ? 2 * nb : 0; }
FCPB_DEV int q_num_blocks(const QRef& qr) { return (qr.q_len + kBQ - 1) / kBQ; }

// 4-byte async copy with zero fill when !valid; completion tracked by an mbarrier.
FCPB_DEV void cp_async_4(void* smem_dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
               ::"r"(smem_u32(smem_dst)), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
FCPB_DEV void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 64 columns (two x32 loads), waits for completion.
FCPB_DEV void tmem_ld64(uint32_t taddr, float (&out)[64]) {
  uint32_t a[32], b[32];
  tmem_ld32(taddr, a);
  tmem_ld32(taddr + 32, b);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    out[i] = __uint_as_float(a[i]);
    out[32 + i] = __uint_as_float(b[i]);
  }
}

FCPB_DEV float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// One kv row of one Q tile:  P = exp2(S*c + nlse2[q]),  dS = P (dP + ndelta[q]), packed to
// bf16 pairs in TMEM (32 columns each: the A operands of the dV / dK matmuls).
// nlse2 = -lse*log2(e), ndelta = -delta (preprocess).
// kMask: ragged kv row / ragged q columns / causal diagonal (col >= shift) masking.
template <bool kMask>
FCPB_DEV void softmax_half(const uint32_t (&s)[32], const uint32_t (&dp)[32], uint32_t l2,
                           uint32_t dl, float sl2, uint32_t t_p, uint32_t t_ds, bool kv_live,
                           int q_valid, int shift, int half) {
  const float2 c2 = make_float2(sl2, sl2);
  uint32_t pk[16], dk[16];
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8) {
    const int cb = half * 32 + c8 * 8;
    const float4 la = lds128(l2 + cb * 4), lb = lds128(l2 + cb * 4 + 16);
    const float4 da = lds128(dl + cb * 4), dbv = lds128(dl + cb * 4 + 16);
    const float2 nl[4] = {make_float2(la.x, la.y), make_float2(la.z, la.w), make_float2(lb.x, lb.y),
                          make_float2(lb.z, lb.w)};
    const float2 nd[4] = {make_float2(da.x, da.y), make_float2(da.z, da.w),
                          make_float2(dbv.x, dbv.y), make_float2(dbv.z, dbv.w)};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = c8 * 8 + 2 * u;
      const int col = half * 32 + i;
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), c2, nl[u]);
      float p0 = ex2(x.x), p1 = ex2(x.y);
      if (kMask) {
        p0 = (kv_live && col < q_valid && col >= shift) ? p0 : 0.f;
        p1 = (kv_live && col + 1 < q_valid && col + 1 >= shift) ? p1 : 0.f;
      }
      const float2 pp = make_float2(p0, p1);
      const float2 dd = __fmul2_rn(
          pp, __fadd2_rn(make_float2(__uint_as_float(dp[i]), __uint_as_float(dp[i + 1])), nd[u]));
      pk[c8 * 4 + u] = pack_bf16(pp.x, pp.y);
      dk[c8 * 4 + u] = pack_bf16(dd.x, dd.y);
    }
  }
  tmem_st16(t_p + half * 16, pk);
  tmem_st16(t_ds + half * 16, dk);
}

__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q,      // bf16 [Tq,Hq,D], box (64,1,64)
                const __grid_constant__ CUtensorMap tm_do,     // bf16 [Tq,Hq,D], box (64,1,64)
                const __grid_constant__ CUtensorMap tm_k,      // bf16 [Tkv,Hkv,D], box (64,1,128)
                const __grid_constant__ CUtensorMap tm_v,
                const __grid_constant__ CUtensorMap tm_k_recv,
                const __grid_constant__ CUtensorMap tm_v_recv,
                const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = warp_id();
  const int group = p.num_q_heads / p.num_kv_heads;
  const int total = p.num_items * p.num_kv_heads;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_k_recv);
    tma_prefetch_desc(&tm_v_recv);
  }
  if (warp == 1 && elect_one()) {
    mbar_init(&sm.kv_full, 1);
    mbar_init(&sm.kv_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.qd_full[s], 1 + 32);   // TMA expect_tx arrive + 32 cp.async arrives
      mbar_init(&sm.qd_empty[s], 1);
    }
    mbar_init(&sm.sdp_full, 1);
    mbar_init(&sm.sdp_free, 128);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.pds_full[b], 128);
      mbar_init(&sm.pds_free[b], 1);
    }
    mbar_init(&sm.acc_full, 1);
    mbar_init(&sm.acc_free, 128);
    sched_init(sm.sched, 1 + 8);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (all lanes:
    // lane 0 issues the TMA tiles, every lane copies 2 lse2 + 2 delta values with cp.async)
    const uint32_t lane = lane_id();
    const uint64_t keep = policy_evict_last();
    uint32_t kv_phase = 0, stage = 0, stage_phase = 0;
    int ptile = 0;
    SchedCursor sc;
    for (int g; (g = __shfl_sync(0xffffffffu, lane == 0 ? sched_produce(sm.sched, sc, p.sched_counter) : 0, 0)) < total;) {
      const Item it = p.items[item_of(g, p)];
      const int kvh = head_of(g, p);
      const KvSeg ks = p.kvsegs[it.kvseg];
      const bool recv = ks.flags & FCPB_KV_RECV;
      const int krow = ks.kv_off + it.nblock * kBK;
      mbar_wait(&sm.kv_empty, kv_phase ^ 1);
      kv_phase ^= 1;
      if (lane == 0) {
        mbar_arrive_expect_tx(&sm.kv_full, 2 * kKVBytes);
        for (int half = 0; half < 2; ++half) {
          tma_load_3d(&sm.k[half * kKVPanel], recv ? &tm_k_recv : &tm_k, &sm.kv_full, half * 64,
                      kvh, krow);
          tma_load_3d(&sm.v[half * kKVPanel], recv ? &tm_v_recv : &tm_v, &sm.kv_full, half * 64,
                      kvh, krow);
        }
      }
      for (int r = ks.q_begin; r < ks.q_end; ++r) {
        const QRef qr = p.qrefs[r];
        for (int mb = q_first_block(qr, it.nblock); mb < q_num_blocks(qr); ++mb) {
          const int qrow = qr.q_off + mb * kBQ;
          for (int gq = 0; gq < group; ++gq) {
            const int h = kvh * group + gq;
            mbar_wait(&sm.qd_empty[stage], stage_phase ^ 1);
            if (lane == 0) {
              mbar_arrive_expect_tx(&sm.qd_full[stage], 2 * kQBytes);
              for (int half = 0; half < 2; ++half) {
                tma_load_3d_hint(&sm.q[stage][half * kQPanel], &tm_q, &sm.qd_full[stage],
                                 half * 64, h, qrow, keep);
                tma_load_3d_hint(&sm.dout[stage][half * kQPanel], &tm_do, &sm.qd_full[stage],
                                 half * 64, h, qrow, keep);
              }
            }
            const float* lsrc = p.lse2_t + static_cast<int64_t>(h) * p.t_pad + qrow;
            const float* dsrc = p.delta_t + static_cast<int64_t>(h) * p.t_pad + qrow;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int i = lane + 32 * u;
              const bool ok = qrow + i < p.q_tokens;
              cp_async_4(&sm.lse2[stage][i], ok ? lsrc + i : p.lse2_t, ok);
              cp_async_4(&sm.delta[stage][i], ok ? dsrc + i : p.delta_t, ok);
            }
            cp_async_arrive_noinc(&sm.qd_full[stage]);
            FCPB_TR(kTrQdIssue, ptile); ++ptile;
            if (++stage == kStages) { stage = 0; stage_phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t id_sdp = idesc_bf16_f32(kBK, kBQ, false, false);  // S^T, dP^T
    const uint32_t id_acc = idesc_bf16_f32(kBK, kD, false, true);    // dV, dK
    const uint32_t a_k = smem_u32(sm.k), a_v = smem_u32(sm.v);
    const bool leader = elect_one();
    uint32_t kv_phase = 0, stage = 0, stage_phase = 0, sdpf_phase = 0, acc_phase = 0;
    uint32_t pds_phase[2] = {0, 0};
    uint32_t tile = 0;   // running Q-tile counter (selects P/dS and dQ buffers)

    auto issue_sdp = [&](uint32_t st) {
      const uint32_t a_q = smem_u32(sm.q[st]), a_do = smem_u32(sm.dout[st]);
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t oa = (kk >> 2) * kKVPanel + (kk & 3) * 32;
          const uint32_t ob = (kk >> 2) * kQPanel + (kk & 3) * 32;
          mma_ss(tmem + kColS, smem_desc_sw128(a_k + oa, 16, 1024),
                 smem_desc_sw128(a_q + ob, 16, 1024), id_sdp, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t oa = (kk >> 2) * kKVPanel + (kk & 3) * 32;
          const uint32_t ob = (kk >> 2) * kQPanel + (kk & 3) * 32;
          mma_ss(tmem + kColDP, smem_desc_sw128(a_v + oa, 16, 1024),
                 smem_desc_sw128(a_do + ob, 16, 1024), id_sdp, kk > 0);
        }
        mma_commit(&sm.sdp_full);
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
        n += (q_num_blocks(qr) - q_first_block(qr, it.nblock)) * group;
      }
      mbar_wait(&sm.kv_full, kv_phase);
      kv_phase ^= 1;
      // tile 0 of this item: S/dP region must have been read by the previous softmax
      mbar_wait(&sm.qd_full[stage], stage_phase);
      FCPB_TR(kTrQdGot, (int)tile);
      mbar_wait(&sm.sdp_free, sdpf_phase ^ 1);
      sdpf_phase ^= 1;
      tc_fence_after();
      issue_sdp(stage);
      FCPB_TR(kTrSdpIssue, (int)tile);
      uint32_t cur_stage = stage;
      if (++stage == kStages) { stage = 0; stage_phase ^= 1; }
      for (int j = 0; j < n; ++j, ++tile) {
        const uint32_t b = tile & 1;
        const uint32_t st_j = cur_stage;
        if (j + 1 < n) {
          mbar_wait(&sm.qd_full[stage], stage_phase);
          FCPB_TR(kTrQdGot, (int)tile + 1);
          mbar_wait(&sm.sdp_free, sdpf_phase ^ 1);   // softmax(j) has S/dP(j) in registers
          sdpf_phase ^= 1;
          tc_fence_after();
          issue_sdp(stage);
          FCPB_TR(kTrSdpIssue, (int)tile + 1);
          cur_stage = stage;
          if (++stage == kStages) { stage = 0; stage_phase ^= 1; }
        }
        mbar_wait(&sm.pds_full[b], pds_phase[b]);
        pds_phase[b] ^= 1;
        FCPB_TR(kTrPdsGot, (int)tile);
        if (j == 0) {
          mbar_wait(&sm.acc_free, acc_phase ^ 1);
          acc_phase ^= 1;
        }
        tc_fence_after();
        if (leader) {
          const uint32_t a_q = smem_u32(sm.q[st_j]), a_do = smem_u32(sm.dout[st_j]);
#pragma unroll
          for (int kk = 0; kk < kBQ / 16; ++kk)     // dV += P^T dO   (A = P^T in TMEM)
            mma_ts(tmem + kColDV, tmem + col_p(b) + kk * 8,
                   smem_desc_sw128(a_do + kk * 2048, kQPanel, 1024), id_acc, (j > 0 || kk > 0));
#pragma unroll
          for (int kk = 0; kk < kBQ / 16; ++kk)     // dK += dS^T Q   (A = dS^T in TMEM)
            mma_ts(tmem + kColDK, tmem + col_ds(b) + kk * 8,
                   smem_desc_sw128(a_q + kk * 2048, kQPanel, 1024), id_acc, (j > 0 || kk > 0));
          mma_commit(&sm.qd_empty[st_j]);
          mma_commit(&sm.pds_free[b]);
          FCPB_TR(kTrAccIssue, (int)tile);
        }
        __syncwarp();
      }
      if (leader) {
        mma_commit(&sm.acc_full);
        mma_commit(&sm.kv_empty);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ softmax (thread == kv row)
    const int tid = threadIdx.x - 128;
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_bits + kColS;
    const uint32_t t_dp = tmem + lane_bits + kColDP;
    const float sl2 = p.scale_log2;
    const uint32_t t_p[2] = {tmem + lane_bits + col_p(0), tmem + lane_bits + col_p(1)};
    const uint32_t t_ds[2] = {tmem + lane_bits + col_ds(0), tmem + lane_bits + col_ds(1)};
    uint32_t sdp_phase = 0, stage = 0, stage_phase = 0, tile = 0;
    uint32_t pfree_phase[2] = {0, 0};
    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      const Item it = p.items[item_of(g, p)];
      const KvSeg ks = p.kvsegs[it.kvseg];
      const int kv_row = it.nblock * kBK + tid;
      const bool kv_live = kv_row < ks.kv_len;
      const bool kv_full_tile = it.nblock * kBK + kBK <= ks.kv_len;
      for (int r = ks.q_begin; r < ks.q_end; ++r) {
        const QRef qr = p.qrefs[r];
        for (int mb = q_first_block(qr, it.nblock); mb < q_num_blocks(qr); ++mb) {
          const int q_valid = qr.q_len - mb * kBQ;
          // diagonal: column c (q = 64mb + c) sees kv row 128nb + tid iff c >= shift
          const int shift0 = (it.nblock * kBK - mb * kBQ);
          const bool plain = kv_full_tile && q_valid >= kBQ && (!qr.diag || shift0 + kBK - 1 <= 0);
          const int shift = qr.diag ? shift0 + tid : -1;
          for (int gq = 0; gq < group; ++gq, ++tile) {
            const uint32_t b = tile & 1;
            mbar_wait(&sm.sdp_full, sdp_phase);
            FCPB_TR(kTrSdpGot, (int)tile);
            sdp_phase ^= 1;
            mbar_wait(&sm.qd_full[stage], stage_phase);   // lse2 / delta of this tile landed
            tc_fence_after();
            const uint32_t l2 = smem_u32(sm.lse2[stage]);
            const uint32_t dl = smem_u32(sm.delta[stage]);
            mbar_wait(&sm.pds_free[b], pfree_phase[b] ^ 1);   // P/dS buffer b consumed (tile j-2)
            pfree_phase[b] ^= 1;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t sv[32], dv[32];
              tmem_ld32(t_s + half * 32, sv);
              tmem_ld32(t_dp + half * 32, dv);
              tmem_wait_ld();
              if (half == 1) {
                tc_fence_before();
                mbar_arrive(&sm.sdp_free);                  // S/dP(j) fully read
                FCPB_TR(kTrLoaded, (int)tile);
              }
              if (plain)
                softmax_half<false>(sv, dv, l2, dl, sl2, t_p[b], t_ds[b], true, kBQ, -1, half);
              else
                softmax_half<true>(sv, dv, l2, dl, sl2, t_p[b], t_ds[b], kv_live, q_valid, shift, half);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.pds_full[b]);
            FCPB_TR(kTrPdsArrive, (int)tile);
            if (++stage == kStages) { stage = 0; stage_phase ^= 1; }
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ dK/dV epilogue
    const int tid = threadIdx.x - 256;            // kv row
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc_phase = 0;
    SchedCursor sc;
    for (int g; (g = sched_consume(sm.sched, sc)) < total;) {
      const Item it = p.items[item_of(g, p)];
      const int kvh = head_of(g, p);
      const KvSeg ks = p.kvsegs[it.kvseg];
      // ---- dK, dV epilogue (thread == kv row)
      mbar_wait(&sm.acc_full, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      const int kv_row = it.nblock * kBK + tid;
      const bool kv_live = kv_row < ks.kv_len;
      const bool recv = ks.flags & FCPB_KV_RECV;
      float* dkb = recv ? p.dk_recv : p.dk;
      float* dvb = recv ? p.dv_recv : p.dv;
      const size_t row = (static_cast<size_t>(ks.kv_off + kv_row) * p.num_kv_heads + kvh) * kD;
#pragma unroll
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t a[32], bb[32];
        tmem_ld32(tmem + lane_bits + kColDK + c * 32, a);
        tmem_ld32(tmem + lane_bits + kColDV + c * 32, bb);
        tmem_wait_ld();
        if (kv_live) {
          float4* k4 = reinterpret_cast<float4*>(dkb + row + c * 32);
          float4* v4 = reinterpret_cast<float4*>(dvb + row + c * 32);
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
