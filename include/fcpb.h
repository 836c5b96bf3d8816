/*
 * fcpb.h -- C ABI of the B200-native FCP block-attention data plane (libfcpb.so).
 *
 * The reference (arxiv 2605.08524, package `blocksched`) has no FFI: its data
 * plane is the analytic stand-in
 *     simulate(assignment, plan, units, deps, hw, cfg, curve, opts) -> SimReport
 * (reference pkg/src/blocksched/simulator.py:154-232), and attention math exists
 * only in the paper.  These entry points are what a binding of
 * that data plane needs: they *execute* the (Q chunk, KV chunk) tiles of
 * DependencyMap.q_to_kv (reference sharding.py:172-201) that simulate() only
 * times (simulator.py:73-109), merge the per-stage partial outputs, and reduce
 * the dK/dV partials that return along the reversed edges of the plan
 * (planner.py:81-102, reversed).
 *
 * Conventions
 *  - All tensors are dense, token-major: Q/O/dO [T, Hq, D], K/V [T, Hkv, D],
 *    bf16 unless noted; LSE is fp32 [T, Hq], natural log; softmax scale given.
 *  - q-head h uses kv-head h / (Hq/Hkv)  (GQA; the reference leaves this open).
 *  - Every pointer is a device pointer owned by the caller; the library
 *    allocates nothing (except the fcpb_ipc_* transport regions) and never
 *    synchronises on the compute path; `stream` is a cudaStream_t.
 *  - Returns 0 (FCPB_OK) or a negative fcpb_status; fcpb_last_error() gives the
 *    message (thread-local).  Python maps these onto ParameterError / NativeError.
 *  - sm_100a only (B200).  D = 128, Hq/Hkv even for the tcgen05 kernels.
 */
#ifndef FCPB_H_
#define FCPB_H_

#include <stddef.h>
#include <stdint.h>

#include "../paper_2605_08524_b200/csrc/fcpb_types.h"

#if defined(__GNUC__)
#define FCPB_API __attribute__((visibility("default")))
#else
#define FCPB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum fcpb_status {
  FCPB_OK = 0,
  FCPB_ERR_INVALID = -1,   /* bad shape / argument (ParameterError)            */
  FCPB_ERR_CUDA = -2,      /* CUDA runtime / driver failure (NativeError)      */
  FCPB_ERR_UNSUPPORTED = -3 /* device is not sm_100 or shape not compiled     */
};

/* Forward (K1).  Replaces the per-tile compute that simulate() accounts for in
 * _tile_seconds_by_release (simulator.py:73-109). */
typedef struct {
  int32_t num_q_heads, num_kv_heads, head_dim;
  float softmax_scale;
  const void* q;           int64_t q_tokens;          /* [Tq, Hq, D] bf16            */
  const void* k;           const void* v;             /* local KV [Tkv, Hkv, D] bf16 */
  int64_t kv_tokens;
  const void* k_recv;      const void* v_recv;        /* receive arena (may be NULL) */
  int64_t kv_recv_tokens;
  void* o;                 float* lse;                /* final outputs                */
  float* o_partial;        float* lse_partial;        /* [P, Hq, D] / [P, Hq] or NULL */
  int64_t partial_rows;
  const FcpbSegment* segments; int32_t num_segments;  /* device tables (worklist.py) */
  const FcpbKvRef* kv_refs;    int32_t num_kv_refs;
  const FcpbItem* items;       int32_t num_items;     /* LPT-ordered                  */
  int32_t num_ctas;            /* 0 = one per SM                                      */
  int32_t head_major;          /* grid order: 0 = heads of an item adjacent, 1 = items of a head */
  int32_t hm_lead;             /* head_major: the first hm_lead (largest) items still run heads-adjacent */
  int32_t* sched_counter;      /* device int scratch for the dynamic tile scheduler (zeroed here) */
} FcpbFwdArgs;

FCPB_API int fcpb_attn_fwd(const FcpbFwdArgs* args, void* stream);

/* K3: LSE merge of per-stage partial outputs.  Group g covers Q tokens
 * [q_off, q_off+q_len) whose partial rows start at part_rows[part_begin..part_end). */
typedef struct {
  int32_t q_off, q_len, part_begin, part_end;
  int32_t tok_begin;           /* prefix sum of q_len over preceding groups */
  int32_t pad_;
} FcpbMergeGroup;

typedef struct {
  int32_t num_q_heads, head_dim;
  const float* o_partial; const float* lse_partial;
  const FcpbMergeGroup* groups; int32_t num_groups;
  const int32_t* part_rows;
  int64_t merged_tokens;       /* sum of q_len over groups */
  void* o; float* lse;         /* bf16 [Tq,Hq,D], fp32 [Tq,Hq] */
} FcpbMergeArgs;

FCPB_API int fcpb_lse_merge(const FcpbMergeArgs* args, void* stream);

/* K2 preprocess (num_q_heads <= 64): -delta = -rowsum(dO * O) and -lse * log2(e), both written negated and
 * head-major [Hq, t_pad] fp32 (t_pad = tokens rounded up to 4, TMA row pitch), and
 * zero the fp32 dQ accumulator [tokens, Hq, D]. */
FCPB_API int fcpb_bwd_preprocess(const void* o, const void* dout, const float* lse,
                                 float* lse2_t, float* delta_t, int64_t t_pad, float* dq_accum,
                                 int64_t tokens, int32_t num_q_heads, int32_t head_dim,
                                 void* stream);

/* K2b: dQ of the backward, query-stationary (one CTA per 128 query rows x head): the
 * segment / KV-ref / item tables have the forward's layout but each segment lists ALL
 * KV chunks its Q chunk attends to (local and received).  Writes bf16 dQ once
 * (scale applied); needs lse2_t / delta_t from fcpb_bwd_preprocess. */
typedef struct {
  int32_t num_q_heads, num_kv_heads, head_dim;
  float softmax_scale;
  const void* q; const void* dout;
  const float* lse2_t; const float* delta_t; int64_t t_pad;
  int64_t q_tokens;
  const void* k; const void* v; int64_t kv_tokens;
  const void* k_recv; const void* v_recv; int64_t kv_recv_tokens;
  void* dq;                                    /* bf16 [Tq, Hq, D] */
  const FcpbSegment* segments; int32_t num_segments;
  const FcpbKvRef* kv_refs;    int32_t num_kv_refs;
  const FcpbItem* items;       int32_t num_items;
  int32_t num_ctas;
  int32_t head_major;
  int32_t hm_lead;
  int32_t* sched_counter;      /* device int scratch for the dynamic tile scheduler (zeroed here) */
} FcpbDqArgs;

FCPB_API int fcpb_attn_bwd_dq(const FcpbDqArgs* args, void* stream);

/* K2: backward dK/dV.  Work is organised by KV tile: for each KV segment (a local run of
 * chunks, or a group of received chunks back to back in the arena) the list of local Q
 * runs that attend to it.  dK/dV accumulate in fp32 per KV arena row (plain stores: one
 * CTA owns a KV block for all heads of its GQA group). */
typedef struct {
  int32_t kv_off, kv_len;       /* arena rows of the KV segment                     */
  int32_t flags;                /* FCPB_KV_RECV: lives in the receive arena         */
  int32_t q_begin, q_end;       /* [q_begin,q_end) into FcpbBwdQRef                  */
  int32_t pad_;
} FcpbBwdKvSeg;

typedef struct {
  int32_t q_off, q_len;
  int32_t diag;                 /* causal diagonal tile (Q run == KV run)           */
  int32_t kv_limit;             /* 0: every row of the segment is visible; else only
                                   its first kv_limit rows (a received group's prefix
                                   of chunks before this Q run)                     */
} FcpbBwdQRef;

typedef struct {
  int32_t kvseg;                /* FcpbBwdKvSeg index                                */
  int32_t nblock;               /* 128-row KV block inside the chunk                */
} FcpbBwdItem;

typedef struct {
  int32_t num_q_heads, num_kv_heads, head_dim;
  float softmax_scale;
  const void* q; const void* dout;
  const float* lse2_t; const float* delta_t; int64_t t_pad;   /* from fcpb_bwd_preprocess */
  int64_t q_tokens;
  const void* k; const void* v; int64_t kv_tokens;
  const void* k_recv; const void* v_recv; int64_t kv_recv_tokens;
  float* dq_accum;              /* unused (dQ comes from fcpb_attn_bwd_dq); may be NULL */
  float* dk_accum; float* dv_accum;             /* local  [Tkv, Hkv, D] fp32         */
  float* dk_recv_accum; float* dv_recv_accum;   /* recv   [Trecv, Hkv, D] fp32       */
  void* dk_out; void* dv_out;   /* optional bf16 [Tkv, Hkv, D]: local segments write the final
                                   (scaled) dK/dV here instead of dk/dv_accum -- only when no
                                   partials of this rank's chunks come back from peers      */
  void* ds_out;                 /* optional bf16 dS^T tiles [pairs * Hq][128 q / 8][128 kv][8 q] for
                                   fcpb_attn_bwd_dq_ds (materialised-dS backward)         */
  const int32_t* pair_base;     /* with ds_out: per item, its first (kv block, q block) pair */
  const FcpbBwdKvSeg* kvsegs; int32_t num_kvsegs;
  const FcpbBwdQRef* qrefs; int32_t num_qrefs;
  const FcpbBwdItem* items; int32_t num_items;
  int32_t num_ctas;
  int32_t head_major;
  int32_t hm_lead;
  int32_t* sched_counter;      /* device int scratch for the dynamic tile scheduler (zeroed here) */
} FcpbBwdArgs;

FCPB_API int fcpb_attn_bwd(const FcpbBwdArgs* args, void* stream);

/* K2c: dQ from materialised dS tiles (written by fcpb_attn_bwd with ds_out): a grouped
 * GEMM dQ = scale * sum dS K over each item's KV tiles.  Tables as FcpbDqArgs, plus the
 * dS pair id of every (item, KV tile) (worklist.build_ds_tiles). */
typedef struct {
  int32_t num_q_heads, num_kv_heads, head_dim;
  float softmax_scale;
  const void* ds; int64_t ds_tiles;              /* bf16 [ds_tiles][16][128][8] (see ds_out) */
  const void* k; int64_t kv_tokens;
  const void* k_recv; int64_t kv_recv_tokens;
  void* dq;                                      /* bf16 [Tq, Hq, D] output                */
  const FcpbSegment* segments; int32_t num_segments;
  const FcpbKvRef* kv_refs;    int32_t num_kv_refs;
  const FcpbItem* items;       int32_t num_items;
  const int32_t* pair_ids; const int32_t* pair_off;
  int32_t num_ctas;
  int32_t head_major;
  int32_t hm_lead;
  int32_t* sched_counter;
} FcpbDqDsArgs;

FCPB_API int fcpb_attn_bwd_dq_ds(const FcpbDqDsArgs* args, void* stream);

/* fp32 -> bf16 conversion of an accumulator (dQ, dK, dV). */
FCPB_API int fcpb_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream);

/* K4: dK/dV reduce at the owner: dst[rows[i]] += src[i] for `n_rows` rows of
 * `row_elems` fp32 each (partials returned along reversed plan edges). */
FCPB_API int fcpb_dkv_reduce(float* dst, const float* src, const int32_t* dst_rows, int64_t n_rows,
                    int64_t row_elems, void* stream);

/* K4 (fused): the owner's final bf16 dK, dV rows: out[r] = bf16(local[r] + sum of
 * staged[src_rows[j]] for j in [row_ptr[r], row_ptr[r+1])), for `n_rows` rows of `row_elems`
 * fp32.  The staged rows are the partials consumers returned along reversed plan edges; the
 * reference never models this step.  Replaces fcpb_dkv_reduce rounds plus
 * two fcpb_f32_to_bf16 passes. */
FCPB_API int fcpb_dkv_finalize(const float* local_k, const float* local_v, const float* staged_k,
                               const float* staged_v, const int32_t* row_ptr,
                               const int32_t* src_rows, int64_t n_rows, int64_t row_elems,
                               void* out_k, void* out_v, void* stream);

/* Exchange readiness flags without an SM (stream memory operations; replaces a signalling
 * kernel, which cannot become resident beside the persistent attention kernels).
 * fcpb_stream_signal: after the stream's prior work, write `value` to the 32-bit `flag`
 *   (local or peer-mapped symmetric memory), preceded by a stream-scoped system fence.
 * fcpb_stream_wait: later work on the stream waits until (int32)(*flag - value) >= 0.
 * Replaces the symmetric-memory barrier kernels the exchange used around each pull set
 * (the reference models this ordering as stage boundaries, simulator.py:136-151). */
FCPB_API int fcpb_stream_signal(void* flag, uint32_t value, void* stream);
FCPB_API int fcpb_stream_wait(const void* flag, uint32_t value, void* stream);

/* Peer-memory regions for the K5 KV exchange and the K6 dK/dV return (the one place the
 * library allocates, on behalf of the transport): device memory with a CUDA IPC handle that
 * the other ranks (processes) open and copy from with copy-engine memcpys.  Works across the
 * GPUs of one NVSwitch box and between processes that share one GPU.  The reference models
 * this transport only analytically (simulator.py:136-151). */
typedef struct { char reserved[64]; } FcpbIpcHandle;
FCPB_API int fcpb_ipc_alloc(int device, size_t bytes, void** ptr, FcpbIpcHandle* handle);
FCPB_API int fcpb_ipc_open(int device, const FcpbIpcHandle* handle, void** ptr);
FCPB_API int fcpb_ipc_close(int device, void* ptr);
FCPB_API int fcpb_ipc_free(int device, void* ptr);
/* One copy-engine transfer of `height` rows of `width` bytes (pitches in bytes), ordered on
 * `stream`: a run of K rows and the matching V rows (two planes of one region) move as one
 * 2-D copy instead of two. */
FCPB_API int fcpb_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                          size_t height, void* stream);

/* K5 pull kernel: copy `num_segs` byte ranges {dst, src, bytes} (a device array of
 * FcpbGatherSeg; addresses 16-byte aligned, bytes a multiple of 16 and at most
 * fcpb_gather_seg_bytes()) with SM loads -- src typically a peer's IPC region read over
 * NVLink -- on `num_ctas` CTAs.  Used when nothing overlaps the forward pulls (one forward
 * wave after the exchange), where it outruns copy-engine transfers of a few MB each. */
typedef struct { uint64_t dst; uint64_t src; int64_t bytes; } FcpbGatherSeg;
FCPB_API int fcpb_gather_copy(const void* segs, int32_t num_segs, int32_t num_ctas, void* stream);
FCPB_API int64_t fcpb_gather_seg_bytes(void);

/* The same copy with base-relative segments: dst and src of each segment are
 * (base index << 56) | byte offset into bases[index] (num_bases <= FCPB_GATHER_MAX_BASES, the
 * bases passed by value).  A segment table that depends only on a move's shape (the
 * reshuffler's runs) is uploaded once and reused whatever the tensors' addresses are. */
#define FCPB_GATHER_MAX_BASES 32
FCPB_API int fcpb_gather_copy_based(const void* segs, int32_t num_segs, const uint64_t* bases,
                                    int32_t num_bases, int32_t num_ctas, void* stream);

/* Workspace queries: bytes the caller provides for
 *  - the backward preprocess outputs lse2_t + delta_t ([Hq, t_pad] fp32 each, t_pad = T
 *    rounded up to 4);
 *  - the forward partials o_partial [P, Hq, D] fp32 + lse_partial [P, Hq] fp32 of the Q
 *    chunks whose KV list spans several exchange stages (merged by fcpb_lse_merge);
 *  - the materialised-dS tiles (bf16 128x128 per (KV block, Q block, q-head) pair) that
 *    fcpb_attn_bwd writes and fcpb_attn_bwd_dq_ds reads. */
FCPB_API size_t fcpb_bwd_preprocess_bytes(int64_t tokens, int32_t num_q_heads);
FCPB_API size_t fcpb_fwd_partial_bytes(int64_t partial_rows, int32_t num_q_heads, int32_t head_dim);
FCPB_API size_t fcpb_ds_tile_bytes(int64_t ds_pairs, int32_t num_q_heads);

/* Test hook: out[0] = warp-level lazy O-rescale events of fcpb_attn_fwd since the last
 * reset (synchronous; not for the hot path). */
FCPB_API int fcpb_debug_counters(uint64_t* out, int n, int reset);

FCPB_API const char* fcpb_last_error(void);
FCPB_API int fcpb_version(void);
FCPB_API int fcpb_device_supported(int device);

#ifdef __cplusplus
}
#endif
#endif /* FCPB_H_ */
