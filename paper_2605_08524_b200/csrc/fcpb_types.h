// Device-side work-list records shared by the kernels and the C-ABI (plain C layout).
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

// One "segment": a Q chunk together with the ordered run of KV chunks it attends
// to in one launch.  Built on the host from DependencyMap.q_to_kv (worklist.py).
typedef struct {
  int32_t q_off;     // first token of the Q chunk in the rank's packed buffers
  int32_t q_len;     // tokens in the Q chunk
  int32_t kv_begin;  // [kv_begin, kv_end) into the FcpbKvRef array
  int32_t kv_end;
  int32_t out_row;   // -1: write final O/LSE at q_off; >= 0: fp32 partial rows at out_row
  int32_t in_row;    // forward: 0, or 1 + the fp32 partial row block (O, LSE) an earlier wave
                     // wrote for this Q chunk, which this segment continues (no K3 merge)
} FcpbSegment;

// One KV chunk reference.
typedef struct {
  int32_t off;    // first token in its arena (local or receive arena)
  int32_t len;    // tokens
  int32_t flags;  // bit0: causal diagonal tile (KV chunk == Q chunk); bit1: lives in receive arena
  int32_t pad_;
} FcpbKvRef;

#define FCPB_KV_DIAG 1
#define FCPB_KV_RECV 2

// A forward work item: rows [128*mblock, 128*mblock+128) of segment `seg`, all head pairs.
typedef struct {
  int32_t seg;
  int32_t mblock;
} FcpbItem;

#ifdef __cplusplus
}
#endif
