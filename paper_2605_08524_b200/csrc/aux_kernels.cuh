// HBM-bound helper kernels: K3 LSE merge, K2 preprocess, K4 dK/dV reduce, fp32->bf16.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "../../include/fcpb.h"

namespace fcpb {
namespace aux {

// K3: one warp per (merged token, kMergeHeads consecutive q-heads); lane owns 4 of the 128
// head-dim values.  lse = logsumexp_s lse_s ; O = sum_s exp(lse_s - lse) O_s (partials are
// normalised).  The heads of one token share the group lookup and the partial row offsets,
// so the warp pays that dependent chain once and keeps kMergeHeads O rows in flight.
#ifndef FCPB_MERGE_HEADS
#define FCPB_MERGE_HEADS 2
#endif
constexpr int kMergeHeads = FCPB_MERGE_HEADS;
__global__ void __launch_bounds__(256) lse_merge_kernel(const FcpbMergeArgs a) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int H = a.num_q_heads;
  const int hb = (H + kMergeHeads - 1) / kMergeHeads;
  if (w >= a.merged_tokens * hb) return;
  const int tok = static_cast<int>(w / hb);
  const int h0 = static_cast<int>(w % hb) * kMergeHeads;
  int lo = 0, hi = a.num_groups - 1;  // last group with tok_begin <= tok
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.groups[mid].tok_begin <= tok) lo = mid; else hi = mid - 1;
  }
  const FcpbMergeGroup g = a.groups[lo];
  const int t = tok - g.tok_begin;
  float m[kMergeHeads];
#pragma unroll
  for (int u = 0; u < kMergeHeads; ++u) m[u] = -INFINITY;
  for (int s = g.part_begin; s < g.part_end; ++s) {
    const int64_t rb = static_cast<int64_t>(a.part_rows[s] + t) * H + h0;
#pragma unroll
    for (int u = 0; u < kMergeHeads; ++u)
      if (h0 + u < H) m[u] = fmaxf(m[u], a.lse_partial[rb + u]);
  }
  float4 acc[kMergeHeads];
  float wsum[kMergeHeads];
#pragma unroll
  for (int u = 0; u < kMergeHeads; ++u) {
    m[u] = (m[u] == -INFINITY) ? 0.f : m[u];
    acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    wsum[u] = 0.f;
  }
  for (int s = g.part_begin; s < g.part_end; ++s) {
    const int64_t rb = static_cast<int64_t>(a.part_rows[s] + t) * H + h0;
    float4 o[kMergeHeads];
#pragma unroll
    for (int u = 0; u < kMergeHeads; ++u)
      o[u] = h0 + u < H ? reinterpret_cast<const float4*>(a.o_partial + (rb + u) * 128)[lane]
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < kMergeHeads; ++u) {
      const float wt = h0 + u < H ? __expf(a.lse_partial[rb + u] - m[u]) : 0.f;
      acc[u].x += wt * o[u].x; acc[u].y += wt * o[u].y; acc[u].z += wt * o[u].z; acc[u].w += wt * o[u].w;
      wsum[u] += wt;
    }
  }
  const int64_t ob = static_cast<int64_t>(g.q_off + t) * H + h0;
#pragma unroll
  for (int u = 0; u < kMergeHeads; ++u) {
    if (h0 + u >= H) break;
    const float inv = wsum[u] > 0.f ? 1.f / wsum[u] : 0.f;
    __nv_bfloat162 lo2 = __floats2bfloat162_rn(acc[u].x * inv, acc[u].y * inv);
    __nv_bfloat162 hi2 = __floats2bfloat162_rn(acc[u].z * inv, acc[u].w * inv);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo2);
    packed.y = *reinterpret_cast<uint32_t*>(&hi2);
    reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.o) + (ob + u) * 128)[lane] = packed;
    if (lane == 0) a.lse[ob + u] = wsum[u] > 0.f ? m[u] + __logf(wsum[u]) : -INFINITY;
  }
}

// Backward preprocess: -delta = -rowsum(dO * O) and -lse * log2(e), written head-major
// [H, t_pad], and (recompute-dQ mode) dq_accum[row,:] = 0.  A block owns 32 consecutive
// tokens x up to kPrepMaxHeads heads (blockIdx.y picks the head group, so any Hq works):
// half-warps stream the (token, head) rows (256 B of O and of dO each, 16 B per lane), park
// the 32 x heads results in shared memory, and write every head's 32 tokens as one coalesced
// 128 B row (a warp-per-row layout wrote one scattered 4 B word per row and ran at half the
// HBM rate).  C2 size: 170 us, 94% of measured HBM bandwidth (one uint2 per lane, a warp per
// row: 225 us; scripts/micro/prep_ab.py).
#ifndef FCPB_PREP_TOKENS
#define FCPB_PREP_TOKENS 32
#endif
#ifndef FCPB_PREP_U
#define FCPB_PREP_U 2
#endif
constexpr int kPrepTokens = FCPB_PREP_TOKENS;
constexpr int kPrepMaxHeads = 64;
__global__ void __launch_bounds__(256) bwd_preprocess_kernel(const __nv_bfloat16* __restrict__ o,
                                                              const __nv_bfloat16* __restrict__ dout,
                                                              const float* __restrict__ lse,
                                                              float* __restrict__ lse2_t,
                                                              float* __restrict__ delta_t,
                                                              int64_t t_pad, float* __restrict__ dq,
                                                              int64_t tokens, int heads) {
  __shared__ float sd[kPrepMaxHeads][kPrepTokens + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kPrepTokens;
  const int nt = static_cast<int>(tokens - t0 < kPrepTokens ? tokens - t0 : kPrepTokens);
  const int h0 = blockIdx.y * kPrepMaxHeads;
  const int hc = heads - h0 < kPrepMaxHeads ? heads - h0 : kPrepMaxHeads;   // heads of this block
  const int nrows = nt * hc;
  constexpr int kU = FCPB_PREP_U;           // row pairs in flight per warp
  // Row r of the block is (token t0 + r / hc, head h0 + r % hc); with hc == heads the rows
  // are contiguous.  A half-warp reads one 256 B row as 16 B per lane, so one warp load
  // covers two rows.
  const int half = lane >> 4, hl = lane & 15;
  auto row_of = [&](int r) -> int64_t {
    return (t0 + r / hc) * heads + h0 + r % hc;
  };
  for (int r0 = warp * 2 * kU; r0 < nrows; r0 += nwarps * 2 * kU) {
    uint4 ov[kU], dv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int r = r0 + 2 * u + half;
      ov[u] = r < nrows ? reinterpret_cast<const uint4*>(o + row_of(r) * 128)[hl] : make_uint4(0, 0, 0, 0);
      dv[u] = r < nrows ? reinterpret_cast<const uint4*>(dout + row_of(r) * 128)[hl] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int r = r0 + 2 * u + half;
      const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov[u]);
      const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv[u]);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(o2[i]);
        const float2 y = __bfloat1622float2(d2[i]);
        s = fmaf(x.x, y.x, s);
        s = fmaf(x.y, y.y, s);
      }
#pragma unroll
      for (int off = 8; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (r < nrows) {
        if (hl == 0) sd[r % hc][r / hc] = -s;
        if (dq) {
          float4* row = reinterpret_cast<float4*>(dq + row_of(r) * 128);
          row[hl] = make_float4(0.f, 0.f, 0.f, 0.f);
          row[hl + 16] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  __syncthreads();
  for (int h = warp; h < hc; h += nwarps) {
    for (int i = lane; i < nt; i += 32) {
      delta_t[(h0 + h) * t_pad + t0 + i] = sd[h][i];
      lse2_t[(h0 + h) * t_pad + t0 + i] = -lse[(t0 + i) * heads + h0 + h] * 1.4426950408889634f;
    }
  }
}

__global__ void __launch_bounds__(256) f32_to_bf16_kernel(const float4* __restrict__ src,
                                                           uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = src[i];
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 r;
    r.x = *reinterpret_cast<uint32_t*>(&lo);
    r.y = *reinterpret_cast<uint32_t*>(&hi);
    dst[i] = r;
  }
}

// K4: dst row dst_rows[i] += src row i (rows of `row4` float4).
__global__ void __launch_bounds__(256) dkv_reduce_kernel(float4* __restrict__ dst,
                                                          const float4* __restrict__ src,
                                                          const int32_t* __restrict__ dst_rows,
                                                          int64_t n_rows, int64_t row4) {
  const int64_t work = n_rows * row4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < work;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / row4, c = i % row4;
    const float4 s = src[i];
    float4& d = dst[static_cast<int64_t>(dst_rows[r]) * row4 + c];
    d.x += s.x; d.y += s.y; d.z += s.z; d.w += s.w;
  }
}

// K4 (fused): the owner's final dK and dV in one pass.  Row r of `local` plus every returned
// partial of it (staging rows src_rows[row_ptr[r] .. row_ptr[r+1]), one per consuming rank),
// rounded once to bf16.  Each output row has one owner thread per float4, so no rounds and
// no atomics; replaces (gather + K4 add) per receiver round and the two fp32->bf16 passes.
__global__ void __launch_bounds__(256) dkv_finalize_kernel(
    const float4* __restrict__ local_k, const float4* __restrict__ local_v,
    const float4* __restrict__ staged_k, const float4* __restrict__ staged_v,
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ src_rows,
    int64_t n_rows, int64_t row4, uint2* __restrict__ out_k, uint2* __restrict__ out_v) {
  const int64_t work = n_rows * row4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < work;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / row4, c = i % row4;
    float4 a = local_k[i], b = local_v[i];
    const int32_t e = row_ptr[r + 1];
    for (int32_t j = row_ptr[r]; j < e; ++j) {
      const int64_t sidx = static_cast<int64_t>(src_rows[j]) * row4 + c;
      const float4 sk = staged_k[sidx], sv = staged_v[sidx];
      a.x += sk.x; a.y += sk.y; a.z += sk.z; a.w += sk.w;
      b.x += sv.x; b.y += sv.y; b.z += sv.z; b.w += sv.w;
    }
    __nv_bfloat162 k0 = __floats2bfloat162_rn(a.x, a.y), k1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 v0 = __floats2bfloat162_rn(b.x, b.y), v1 = __floats2bfloat162_rn(b.z, b.w);
    out_k[i] = make_uint2(*reinterpret_cast<uint32_t*>(&k0), *reinterpret_cast<uint32_t*>(&k1));
    out_v[i] = make_uint2(*reinterpret_cast<uint32_t*>(&v0), *reinterpret_cast<uint32_t*>(&v1));
  }
}

}  // namespace aux
}  // namespace fcpb
