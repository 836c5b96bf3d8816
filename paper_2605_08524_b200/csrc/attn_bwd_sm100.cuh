// K2: varlen block-pair attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// Work item = one 128-row KV block of one KV chunk (local or received) for one
// KV head.  The CTA loops over every (Q chunk, 128-row Q block, q-head of the
// GQA group) that attends to it, so dK/dV accumulate in TMEM without atomics and
// are written exactly once; dQ partials are added into an fp32 accumulator.
//
// Per Q tile j (all matmuls 128x128x128, bf16 in, fp32 accumulate):
//   S^T  = K  Q_j^T      (SS)   -> TMEM [0,128)
//   dP^T = V  dO_j^T     (SS)   -> TMEM [128,256)
//   softmax warps (thread == kv row):  P^T = exp2(S^T*c - lse2[q]),
//        dS^T = P^T (dP^T - delta[q]);  P^T (bf16) -> TMEM [0,64),
//        dS^T (bf16) -> TMEM [128,192) and -> smem (MN-major, A of the dQ matmul)
//   dV  += P^T  dO_j     (TS)   TMEM [256,384)
//   dK  += dS^T Q_j      (TS)   TMEM [384,512)
//   dQ_j = dS   K        (SS)   -> TMEM [128,256), drained with fp32 reductions
// Warps: w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 softmax / dQ drain / dK,dV epilogue.
#pragma once
#include "fcpb_types.h"
#include "sm100_ptx.cuh"

namespace fcpb {
namespace bwd {

constexpr int kD = 128;
constexpr int kB = 128;                    // rows per Q tile and per KV tile
constexpr int kTileBytes = kB * kD * 2;    // 32 KB
constexpr int kHalfBytes = kTileBytes / 2;
constexpr int kStages = 2;                 // (Q, dO) double buffer
constexpr int kThreads = 256;
constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 384;

struct KvSeg {      // mirrors FcpbBwdKvSeg
  int32_t kv_off, kv_len, flags, q_begin, q_end, pad_;
};
struct QRef {       // mirrors FcpbBwdQRef
  int32_t q_off, q_len, diag, pad_;
};
struct Item {       // mirrors FcpbBwdItem
  int32_t kvseg, nblock;
};

struct Smem {
  uint8_t k[kTileBytes];
  uint8_t v[kTileBytes];
  uint8_t q[kStages][kTileBytes];
  uint8_t dout[kStages][kTileBytes];
  uint8_t ds[kTileBytes];          // dS as the MN-major A operand of dQ = dS K
  float lse2[kB];                  // lse * log2(e) of the current Q tile
  float delta[kB];
  uint64_t kv_full, kv_empty;
  uint64_t qd_full[kStages], qd_empty[kStages];
  uint64_t s_full, p_full, dq_full, dq_empty, acc_full, acc_empty;
  uint32_t tmem_base;
};

struct Params {
  const KvSeg* kvsegs;
  const QRef* qrefs;
  const Item* items;
  int32_t num_items;
  int32_t num_q_heads, num_kv_heads;
  float scale;            // softmax scale
  float scale_log2;       // scale * log2(e)
  const float* lse;       // [Tq, Hq] natural log
  const float* delta;     // [Tq, Hq]
  float* dq;              // [Tq, Hq, D] fp32 accumulate
  float* dk;              // local  [Tkv, Hkv, D] fp32
  float* dv;
  float* dk_recv;         // recv   [Tr, Hkv, D] fp32
  float* dv_recv;
};

// Q blocks of `qr` that see KV block `nb`: causal diagonal -> mb >= nb.
FCPB_DEV int q_first_block(const QRef& qr, int nb) { return qr.diag ? nb : 0; }
FCPB_DEV int q_num_blocks(const QRef& qr) { return (qr.q_len + kB - 1) / kB; }

FCPB_DEV void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
               ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_do,
                const __grid_constant__ CUtensorMap tm_k,
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
      mbar_init(&sm.qd_full[s], 1);
      mbar_init(&sm.qd_empty[s], 1);
    }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.p_full, 128);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_empty, 128);
    mbar_init(&sm.acc_full, 1);
    mbar_init(&sm.acc_empty, 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      uint32_t kv_phase = 0, stage = 0, stage_phase = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const Item it = p.items[g / p.num_kv_heads];
        const int kvh = g % p.num_kv_heads;
        const KvSeg ks = p.kvsegs[it.kvseg];
        const bool recv = ks.flags & FCPB_KV_RECV;
        const int krow = ks.kv_off + it.nblock * kB;
        mbar_wait(&sm.kv_empty, kv_phase ^ 1);
        kv_phase ^= 1;
        mbar_arrive_expect_tx(&sm.kv_full, 2 * kTileBytes);
        for (int half = 0; half < 2; ++half) {
          tma_load_3d(&sm.k[half * kHalfBytes], recv ? &tm_k_recv : &tm_k, &sm.kv_full,
                      half * 64, kvh, krow);
          tma_load_3d(&sm.v[half * kHalfBytes], recv ? &tm_v_recv : &tm_v, &sm.kv_full,
                      half * 64, kvh, krow);
        }
        for (int r = ks.q_begin; r < ks.q_end; ++r) {
          const QRef qr = p.qrefs[r];
          for (int mb = q_first_block(qr, it.nblock); mb < q_num_blocks(qr); ++mb) {
            for (int gq = 0; gq < group; ++gq) {
              const int h = kvh * group + gq;
              mbar_wait(&sm.qd_empty[stage], stage_phase ^ 1);
              mbar_arrive_expect_tx(&sm.qd_full[stage], 2 * kTileBytes);
              const int qrow = qr.q_off + mb * kB;
              for (int half = 0; half < 2; ++half) {
                tma_load_3d_hint(&sm.q[stage][half * kHalfBytes], &tm_q, &sm.qd_full[stage],
                                 half * 64, h, qrow, keep);
                tma_load_3d_hint(&sm.dout[stage][half * kHalfBytes], &tm_do, &sm.qd_full[stage],
                                 half * 64, h, qrow, keep);
              }
              if (++stage == kStages) { stage = 0; stage_phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t id_kmaj = idesc_bf16_f32(kB, kB, false, false);  // S^T, dP^T
    const uint32_t id_bmn = idesc_bf16_f32(kB, kD, false, true);    // dV, dK (TS)
    const uint32_t id_dq = idesc_bf16_f32(kB, kD, true, true);      // dQ: A=dS MN-major
    const uint32_t a_k = smem_u32(sm.k), a_v = smem_u32(sm.v), a_ds = smem_u32(sm.ds);
    const bool leader = elect_one();
    uint32_t kv_phase = 0, stage = 0, stage_phase = 0, p_phase = 0, dqe_phase = 0,
             acce_phase = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const Item it = p.items[g / p.num_kv_heads];
      const KvSeg ks = p.kvsegs[it.kvseg];
      mbar_wait(&sm.kv_full, kv_phase);
      kv_phase ^= 1;
      mbar_wait(&sm.acc_empty, acce_phase ^ 1);
      acce_phase ^= 1;
      tc_fence_after();
      int j = 0;
      for (int r = ks.q_begin; r < ks.q_end; ++r) {
        const QRef qr = p.qrefs[r];
        for (int mb = q_first_block(qr, it.nblock); mb < q_num_blocks(qr); ++mb) {
          for (int gq = 0; gq < group; ++gq, ++j) {
            mbar_wait(&sm.qd_full[stage], stage_phase);
            tc_fence_after();
            const uint32_t a_q = smem_u32(sm.q[stage]), a_do = smem_u32(sm.dout[stage]);
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < kD / 16; ++kk) {
                const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
                mma_ss(tmem + kColS, smem_desc_sw128(a_k + off, 16, 1024),
                       smem_desc_sw128(a_q + off, 16, 1024), id_kmaj, kk > 0);
              }
            }
            __syncwarp();
            mbar_wait(&sm.dq_empty, dqe_phase ^ 1);
            dqe_phase ^= 1;
            tc_fence_after();
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < kD / 16; ++kk) {
                const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
                mma_ss(tmem + kColDP, smem_desc_sw128(a_v + off, 16, 1024),
                       smem_desc_sw128(a_do + off, 16, 1024), id_kmaj, kk > 0);
              }
              mma_commit(&sm.s_full);
            }
            __syncwarp();
            mbar_wait(&sm.p_full, p_phase);
            p_phase ^= 1;
            tc_fence_after();
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < kB / 16; ++kk)   // dV += P^T dO
                mma_ts(tmem + kColDV, tmem + kColS + kk * 8,
                       smem_desc_sw128(a_do + kk * 2048, kHalfBytes, 1024), id_bmn,
                       (j > 0 || kk > 0));
#pragma unroll
              for (int kk = 0; kk < kB / 16; ++kk)   // dK += dS^T Q
                mma_ts(tmem + kColDK, tmem + kColDP + kk * 8,
                       smem_desc_sw128(a_q + kk * 2048, kHalfBytes, 1024), id_bmn,
                       (j > 0 || kk > 0));
#pragma unroll
              for (int kk = 0; kk < kB / 16; ++kk)   // dQ = dS K
                mma_ss(tmem + kColDP, smem_desc_sw128(a_ds + kk * 2048, kHalfBytes, 1024),
                       smem_desc_sw128(a_k + kk * 2048, kHalfBytes, 1024), id_dq, kk > 0);
              mma_commit(&sm.dq_full);
              mma_commit(&sm.qd_empty[stage]);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; stage_phase ^= 1; }
          }
        }
      }
      if (leader) {
        mma_commit(&sm.acc_full);
        mma_commit(&sm.kv_empty);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / drains
    const int tid = threadIdx.x - 128;            // 0..127 == TMEM lane
    const uint32_t lane_bits = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_bits + kColS;
    const uint32_t t_dp = tmem + lane_bits + kColDP;
    const uint32_t ds_row = smem_u32(sm.ds) + (tid >> 3) * 1024 + (tid & 7) * 128;
    const float sl2 = p.scale_log2;
    constexpr float kLog2e = 1.4426950408889634f;
    uint32_t s_phase = 0, dq_phase = 0, acc_phase = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const Item it = p.items[g / p.num_kv_heads];
      const int kvh = g % p.num_kv_heads;
      const KvSeg ks = p.kvsegs[it.kvseg];
      const int kv_row = it.nblock * kB + tid;              // row inside the KV chunk
      const bool kv_live = kv_row < ks.kv_len;
      for (int r = ks.q_begin; r < ks.q_end; ++r) {
        const QRef qr = p.qrefs[r];
        for (int mb = q_first_block(qr, it.nblock); mb < q_num_blocks(qr); ++mb) {
          for (int gq = 0; gq < group; ++gq) {
            const int h = kvh * group + gq;
            // per-column statistics of this Q tile
            named_bar_sync(1, 128);
            {
              const int q = mb * kB + tid;
              float l2 = 0.f, dl = 0.f;
              if (q < qr.q_len) {
                const size_t idx = static_cast<size_t>(qr.q_off + q) * p.num_q_heads + h;
                l2 = p.lse[idx] * kLog2e;
                dl = p.delta[idx];
              }
              sm.lse2[tid] = l2;
              sm.delta[tid] = dl;
            }
            named_bar_sync(1, 128);
            mbar_wait(&sm.s_full, s_phase);
            s_phase ^= 1;
            tc_fence_after();
            const int q_valid = qr.q_len - mb * kB;            // columns < q_valid are live
            // diagonal: column c (q row mb*128+c) sees kv row nb*128+tid iff q >= kv
            const int diag_shift = qr.diag ? (it.nblock - mb) * kB + tid : -1;
#pragma unroll
            for (int c = 0; c < kB / 32; ++c) {
              uint32_t sv[32], dv[32];
              tmem_ld32(t_s + c * 32, sv);
              tmem_ld32(t_dp + c * 32, dv);
              tmem_wait_ld();
              uint32_t pk[16], dk[16];
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float pp[2], dd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int col = c * 32 + i + u;
                  const bool vis = kv_live && col < q_valid && col >= diag_shift;
                  const float pv = vis ? ex2(fmaf(__uint_as_float(sv[i + u]), sl2, -sm.lse2[col])) : 0.f;
                  pp[u] = pv;
                  dd[u] = pv * (__uint_as_float(dv[i + u]) - sm.delta[col]);
                }
                pk[i / 2] = pack_bf16(pp[0], pp[1]);
                dk[i / 2] = pack_bf16(dd[0], dd[1]);
              }
              tmem_st16(t_s + c * 16, pk);
              tmem_st16(t_dp + c * 16, dk);
              // dS^T row `tid`, q columns [32c, 32c+32): 64 bytes into the 128-B row of
              // M-atom (c>>1), 16-B chunks XOR-swizzled by (tid & 7).
              const uint32_t atom = ds_row + (c >> 1) * (kB / 8) * 1024;
#pragma unroll
              for (int ch = 0; ch < 4; ++ch) {
                const uint32_t chunk = ((c & 1) * 4 + ch) ^ (tid & 7);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};"
                             ::"r"(atom + chunk * 16), "r"(dk[ch * 4]), "r"(dk[ch * 4 + 1]),
                               "r"(dk[ch * 4 + 2]), "r"(dk[ch * 4 + 3]) : "memory");
              }
            }
            tmem_wait_st();
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(&sm.p_full);
            // ---- drain dQ_j (thread == q row of the tile)
            mbar_wait(&sm.dq_full, dq_phase);
            dq_phase ^= 1;
            tc_fence_after();
            const bool q_live = tid < q_valid;
            float* dst = p.dq + (static_cast<size_t>(qr.q_off + mb * kB + tid) * p.num_q_heads + h) * kD;
#pragma unroll
            for (int c = 0; c < kD / 32; ++c) {
              uint32_t v[32];
              tmem_ld32(t_dp + c * 32, v);
              tmem_wait_ld();
              if (q_live) {
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                  red_add_v4(dst + c * 32 + i, __uint_as_float(v[i]) * p.scale,
                             __uint_as_float(v[i + 1]) * p.scale, __uint_as_float(v[i + 2]) * p.scale,
                             __uint_as_float(v[i + 3]) * p.scale);
              }
            }
            tc_fence_before();
            mbar_arrive(&sm.dq_empty);
          }
        }
      }
      // ---- dK, dV epilogue (thread == kv row)
      mbar_wait(&sm.acc_full, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      const bool recv = ks.flags & FCPB_KV_RECV;
      float* dkb = recv ? p.dk_recv : p.dk;
      float* dvb = recv ? p.dv_recv : p.dv;
      const size_t row = (static_cast<size_t>(ks.kv_off + kv_row) * p.num_kv_heads + kvh) * kD;
#pragma unroll
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t a[32], b[32];
        tmem_ld32(tmem + lane_bits + kColDK + c * 32, a);
        tmem_ld32(tmem + lane_bits + kColDV + c * 32, b);
        tmem_wait_ld();
        if (kv_live) {
          float4* k4 = reinterpret_cast<float4*>(dkb + row + c * 32);
          float4* v4 = reinterpret_cast<float4*>(dvb + row + c * 32);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            k4[i / 4] = make_float4(__uint_as_float(a[i]) * p.scale, __uint_as_float(a[i + 1]) * p.scale,
                                    __uint_as_float(a[i + 2]) * p.scale, __uint_as_float(a[i + 3]) * p.scale);
            v4[i / 4] = make_float4(__uint_as_float(b[i]), __uint_as_float(b[i + 1]),
                                    __uint_as_float(b[i + 2]), __uint_as_float(b[i + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.acc_empty);
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
