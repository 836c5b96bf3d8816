// libfcpb.so: C ABI over the sm_100a FCP block-attention kernels (see include/fcpb.h).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/fcpb.h"
#include "attn_bwd_sm100.cuh"
#include "attn_dq_sm100.cuh"
#include "attn_dqg_sm100.cuh"
#include "attn_fwd_sm100.cuh"
#include "aux_kernels.cuh"
#include "p2p_kernels.cuh"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define FCPB_CUDA(expr)                                                              \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(FCPB_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                  __FILE__, __LINE__);                                               \
  } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Token-major [T, H, d] tensor -> 3-D map (d, head, token) with box (box_d, 1, box_rows).
int make_map(CUtensorMap* m, const void* base, int64_t tokens, int heads, int d, int box_rows,
             bool fp32 = false, int box_d = 64, bool swizzle = true) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(FCPB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return fail(FCPB_ERR_INVALID, "tensor base must be 16-byte aligned");
  const int esz = fp32 ? 4 : 2;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(heads),
                              static_cast<cuuint64_t>(tokens > 0 ? tokens : 1)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * esz,
                                 static_cast<cuuint64_t>(heads) * d * esz};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_d), 1, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FCPB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FCPB_OK;
}

// Stacked ragged tails (two q-heads per 128-row tile when a Q block has <= 64 rows): on by
// default; FCPB_FWD_STACK=0 / FCPB_BWD_STACK=0 turn off the forward / the backward (dK/dV and
// the dQ GEMM, which must agree on it).
bool env_on(const char* name) {
  const char* e = getenv(name);
  return !(e && e[0] == '0');
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

constexpr size_t kFwdSmem = sizeof(fcpb::fwd::Smem) + 1024;
// K2's rings fill shared memory to within a few hundred bytes of the 227 KB limit, so it gets
// the alignment slack that is left: the dynamic window starts 1024-aligned on sm_100 (after
// the 1 KB system reservation), and the kernel traps if it ever does not.
constexpr size_t kBwdSmem = sizeof(fcpb::bwd::Smem) + 1024 <= 232448 ? sizeof(fcpb::bwd::Smem) + 1024 : 232448;
constexpr size_t kDqSmem = sizeof(fcpb::dq::Smem) + 1024;
constexpr size_t kDqgSmem = sizeof(fcpb::dqg::Smem) + 1024;
static_assert(kDqgSmem <= 232448, "dqg smem budget");
static_assert(kDqSmem <= 232448, "dq smem budget");
static_assert(kFwdSmem <= 232448, "fwd smem budget");
static_assert(kBwdSmem <= 232448, "bwd smem budget");

// cudaFuncAttributeMaxDynamicSharedMemorySize is per device (context): remember, per kernel,
// the devices it has been set on (bit d), so a process that drives several GPUs sets it on
// each.  Racing threads at worst both set it, which is harmless.
int ensure_smem(const void* kernel, size_t bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  FCPB_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = dev < 64 ? (uint64_t{1} << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return FCPB_OK;
  FCPB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.fetch_or(bit, std::memory_order_release);
  return FCPB_OK;
}

std::atomic<uint64_t> g_attr_fwd{0}, g_attr_bwd{0}, g_attr_dq{0}, g_attr_dqg{0};

}  // namespace

extern "C" {

const char* fcpb_last_error(void) { return g_err; }
int fcpb_version(void) { return 1; }

int fcpb_device_supported(int device) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess)
    return 0;
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  return major == 10 && minor == 0;
}

int fcpb_attn_fwd(const FcpbFwdArgs* a, void* stream) {
  if (!a) return fail(FCPB_ERR_INVALID, "null args");
  if (a->head_dim != 128) return fail(FCPB_ERR_UNSUPPORTED, "head_dim %d (need 128)", a->head_dim);
  if (a->num_q_heads % 2 || a->num_kv_heads <= 0 || a->num_q_heads % a->num_kv_heads ||
      (a->num_q_heads / a->num_kv_heads) % 2)
    return fail(FCPB_ERR_UNSUPPORTED, "need Hq/Hkv even (Hq=%d Hkv=%d)", a->num_q_heads,
                a->num_kv_heads);
  if (a->num_items <= 0) return FCPB_OK;
  CUtensorMap tq, tq64, tk, tv, tkr, tvr;
  int rc;
  if ((rc = make_map(&tq, a->q, a->q_tokens, a->num_q_heads, 128, 128))) return rc;
  if ((rc = make_map(&tq64, a->q, a->q_tokens, a->num_q_heads, 128, fcpb::fwd::kStackRows))) return rc;
  if ((rc = make_map(&tk, a->k, a->kv_tokens, a->num_kv_heads, 128, 128))) return rc;
  if ((rc = make_map(&tv, a->v, a->kv_tokens, a->num_kv_heads, 128, 128))) return rc;
  const bool has_recv = a->k_recv && a->v_recv && a->kv_recv_tokens > 0;
  if ((rc = make_map(&tkr, has_recv ? a->k_recv : a->k, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     a->num_kv_heads, 128, 128)))
    return rc;
  if ((rc = make_map(&tvr, has_recv ? a->v_recv : a->v, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     a->num_kv_heads, 128, 128)))
    return rc;
  fcpb::fwd::Params p;
  p.segs = a->segments;
  p.kvrefs = a->kv_refs;
  p.items = a->items;
  p.num_items = a->num_items;
  p.num_q_heads = a->num_q_heads;
  p.num_kv_heads = a->num_kv_heads;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  p.o = static_cast<__nv_bfloat16*>(a->o);
  p.lse = a->lse;
  p.o_part = a->o_partial;
  p.lse_part = a->lse_partial;
  p.head_major = a->head_major;
  p.hm_lead = a->hm_lead;
  // stacked tails need four q-heads per KV head
  static const bool stack_env = env_on("FCPB_FWD_STACK");
  p.stack_tails = stack_env && (a->num_q_heads / a->num_kv_heads) % 4 == 0;
  if (!a->sched_counter) return fail(FCPB_ERR_INVALID, "sched_counter is required");
  p.sched_counter = a->sched_counter;
  FCPB_CUDA(cudaMemsetAsync(a->sched_counter, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
  if ((rc = ensure_smem(reinterpret_cast<const void*>(&fcpb::fwd::attn_fwd_kernel), kFwdSmem, g_attr_fwd)))
    return rc;
  const int total = a->num_items * (a->num_q_heads / 2);
  int grid = a->num_ctas > 0 ? a->num_ctas : sm_count();
  if (grid > total) grid = total;
  fcpb::fwd::attn_fwd_kernel<<<grid, fcpb::fwd::kThreads, kFwdSmem,
                               static_cast<cudaStream_t>(stream)>>>(tq, tq64, tk, tv, tkr, tvr, p);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_attn_bwd(const FcpbBwdArgs* a, void* stream) {
  if (!a) return fail(FCPB_ERR_INVALID, "null args");
  if (a->head_dim != 128) return fail(FCPB_ERR_UNSUPPORTED, "head_dim %d (need 128)", a->head_dim);
  if (a->num_kv_heads <= 0 || a->num_q_heads % a->num_kv_heads)
    return fail(FCPB_ERR_UNSUPPORTED, "Hq %% Hkv != 0");
  if (a->num_items <= 0) return FCPB_OK;
  CUtensorMap tq, tdo, tq64, tdo64, tk, tv, tkr, tvr;
  int rc;
  const int H = a->num_q_heads, Hk = a->num_kv_heads;
  if ((rc = make_map(&tq, a->q, a->q_tokens, H, 128, fcpb::bwd::kBQ))) return rc;
  if ((rc = make_map(&tdo, a->dout, a->q_tokens, H, 128, fcpb::bwd::kBQ))) return rc;
  if ((rc = make_map(&tq64, a->q, a->q_tokens, H, 128, fcpb::bwd::kStackRows))) return rc;
  if ((rc = make_map(&tdo64, a->dout, a->q_tokens, H, 128, fcpb::bwd::kStackRows))) return rc;
  if ((rc = make_map(&tk, a->k, a->kv_tokens, Hk, 128, fcpb::bwd::kBK))) return rc;
  if ((rc = make_map(&tv, a->v, a->kv_tokens, Hk, 128, fcpb::bwd::kBK))) return rc;
  const bool has_recv = a->k_recv && a->v_recv && a->kv_recv_tokens > 0;
  if ((rc = make_map(&tkr, has_recv ? a->k_recv : a->k, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     Hk, 128, fcpb::bwd::kBK)))
    return rc;
  if ((rc = make_map(&tvr, has_recv ? a->v_recv : a->v, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     Hk, 128, fcpb::bwd::kBK)))
    return rc;
  if (a->t_pad < a->q_tokens || !a->lse2_t || !a->delta_t)
    return fail(FCPB_ERR_INVALID, "lse2_t/delta_t/t_pad missing (run fcpb_bwd_preprocess)");
  fcpb::bwd::Params p;
  p.kvsegs = reinterpret_cast<const fcpb::bwd::KvSeg*>(a->kvsegs);
  p.qrefs = reinterpret_cast<const fcpb::bwd::QRef*>(a->qrefs);
  p.items = reinterpret_cast<const fcpb::bwd::Item*>(a->items);
  p.num_items = a->num_items;
  p.num_q_heads = H;
  p.num_kv_heads = Hk;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  p.lse2_t = a->lse2_t;
  p.delta_t = a->delta_t;
  p.t_pad = a->t_pad;
  p.q_tokens = static_cast<int32_t>(a->q_tokens);
  p.head_major = a->head_major;
  p.hm_lead = a->hm_lead;
  p.dk = a->dk_accum;
  p.dv = a->dv_accum;
  p.dk_recv = a->dk_recv_accum;
  p.dv_recv = a->dv_recv_accum;
  p.dk_out = static_cast<__nv_bfloat16*>(a->dk_out);
  p.dv_out = static_cast<__nv_bfloat16*>(a->dv_out);
  p.ds_out = static_cast<__nv_bfloat16*>(a->ds_out);
  p.pair_base = a->pair_base;
  static const bool bwd_stack_env = env_on("FCPB_BWD_STACK");
  p.stack_tails = bwd_stack_env && (H / Hk) % 2 == 0;
  if (p.ds_out && !p.pair_base) return fail(FCPB_ERR_INVALID, "ds_out needs pair_base");
  if (!a->sched_counter) return fail(FCPB_ERR_INVALID, "sched_counter is required");
  p.sched_counter = a->sched_counter;
  FCPB_CUDA(cudaMemsetAsync(a->sched_counter, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
  if ((rc = ensure_smem(reinterpret_cast<const void*>(&fcpb::bwd::attn_bwd_kernel), kBwdSmem, g_attr_bwd)))
    return rc;
  const int total = a->num_items * Hk;
  int grid = a->num_ctas > 0 ? a->num_ctas : sm_count();
  if (grid > total) grid = total;
  fcpb::bwd::attn_bwd_kernel<<<grid, fcpb::bwd::kThreads, kBwdSmem,
                               static_cast<cudaStream_t>(stream)>>>(tq, tdo, tq64, tdo64, tk, tv, tkr, tvr, p);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_attn_bwd_dq(const FcpbDqArgs* a, void* stream) {
  if (!a) return fail(FCPB_ERR_INVALID, "null args");
  if (a->head_dim != 128) return fail(FCPB_ERR_UNSUPPORTED, "head_dim %d (need 128)", a->head_dim);
  if (a->num_kv_heads <= 0 || a->num_q_heads % a->num_kv_heads)
    return fail(FCPB_ERR_UNSUPPORTED, "Hq %% Hkv != 0");
  if (a->num_items <= 0) return FCPB_OK;
  if (a->t_pad < a->q_tokens || !a->lse2_t || !a->delta_t)
    return fail(FCPB_ERR_INVALID, "lse2_t/delta_t/t_pad missing (run fcpb_bwd_preprocess)");
  const int H = a->num_q_heads, Hk = a->num_kv_heads;
  CUtensorMap tk, tv, tkr, tvr;
  int rc;
  if ((rc = make_map(&tk, a->k, a->kv_tokens, Hk, 128, fcpb::dq::kBN))) return rc;
  if ((rc = make_map(&tv, a->v, a->kv_tokens, Hk, 128, fcpb::dq::kBN))) return rc;
  const bool has_recv = a->k_recv && a->v_recv && a->kv_recv_tokens > 0;
  if ((rc = make_map(&tkr, has_recv ? a->k_recv : a->k, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     Hk, 128, fcpb::dq::kBN)))
    return rc;
  if ((rc = make_map(&tvr, has_recv ? a->v_recv : a->v, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     Hk, 128, fcpb::dq::kBN)))
    return rc;
  fcpb::dq::Params p;
  p.segs = a->segments;
  p.kvrefs = a->kv_refs;
  p.items = a->items;
  p.num_items = a->num_items;
  p.num_q_heads = H;
  p.num_kv_heads = Hk;
  p.scale = a->softmax_scale;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  p.lse2_t = a->lse2_t;
  p.delta_t = a->delta_t;
  p.t_pad = a->t_pad;
  p.dq = static_cast<__nv_bfloat16*>(a->dq);
  p.q = static_cast<const __nv_bfloat16*>(a->q);
  p.dout = static_cast<const __nv_bfloat16*>(a->dout);
  p.head_major = a->head_major;
  p.hm_lead = a->hm_lead;
  if (!a->sched_counter) return fail(FCPB_ERR_INVALID, "sched_counter is required");
  p.sched_counter = a->sched_counter;
  FCPB_CUDA(cudaMemsetAsync(a->sched_counter, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
  if ((rc = ensure_smem(reinterpret_cast<const void*>(&fcpb::dq::attn_dq_kernel), kDqSmem, g_attr_dq)))
    return rc;
  const int total = a->num_items * H;
  int grid = a->num_ctas > 0 ? a->num_ctas : sm_count();
  if (grid > total) grid = total;
  fcpb::dq::attn_dq_kernel<<<grid, fcpb::dq::kThreads, kDqSmem, static_cast<cudaStream_t>(stream)>>>(
      tk, tv, tkr, tvr, p);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_attn_bwd_dq_ds(const FcpbDqDsArgs* a, void* stream) {
  if (!a) return fail(FCPB_ERR_INVALID, "null args");
  if (a->head_dim != 128) return fail(FCPB_ERR_UNSUPPORTED, "head_dim %d (need 128)", a->head_dim);
  if (a->num_kv_heads <= 0 || a->num_q_heads % a->num_kv_heads)
    return fail(FCPB_ERR_UNSUPPORTED, "Hq %% Hkv != 0");
  if (a->num_items <= 0) return FCPB_OK;
  if (!a->ds || a->ds_tiles <= 0 || !a->pair_ids || !a->pair_off)
    return fail(FCPB_ERR_INVALID, "dS tiles / pair tables missing");
  const int H = a->num_q_heads, Hk = a->num_kv_heads;
  CUtensorMap tk, tkr;
  int rc;
  if ((rc = make_map(&tk, a->k, a->kv_tokens, Hk, 128, fcpb::dqg::kBN))) return rc;
  const bool has_recv = a->k_recv && a->kv_recv_tokens > 0;
  if ((rc = make_map(&tkr, has_recv ? a->k_recv : a->k, has_recv ? a->kv_recv_tokens : a->kv_tokens,
                     Hk, 128, fcpb::dqg::kBN)))
    return rc;
  fcpb::dqg::Params p;
  p.segs = a->segments;
  p.kvrefs = a->kv_refs;
  p.items = a->items;
  p.ds = static_cast<const __nv_bfloat16*>(a->ds);
  p.pair_ids = a->pair_ids;
  p.pair_off = a->pair_off;
  p.num_items = a->num_items;
  p.num_q_heads = H;
  p.num_kv_heads = Hk;
  p.head_major = a->head_major;
  p.hm_lead = a->hm_lead;
  p.scale = a->softmax_scale;
  p.dq = static_cast<__nv_bfloat16*>(a->dq);
  static const bool dqg_stack_env = env_on("FCPB_BWD_STACK");   // must match fcpb_attn_bwd's tiles
  p.stack_tails = dqg_stack_env && (H / Hk) % 2 == 0;
  if (!a->sched_counter) return fail(FCPB_ERR_INVALID, "sched_counter is required");
  p.sched_counter = a->sched_counter;
  FCPB_CUDA(cudaMemsetAsync(a->sched_counter, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
  if ((rc = ensure_smem(reinterpret_cast<const void*>(&fcpb::dqg::attn_dqg_kernel), kDqgSmem, g_attr_dqg)))
    return rc;
  const int total = a->num_items * H;
  int grid = a->num_ctas > 0 ? a->num_ctas : sm_count();
  if (grid > total) grid = total;
  fcpb::dqg::attn_dqg_kernel<<<grid, fcpb::dqg::kThreads, kDqgSmem, static_cast<cudaStream_t>(stream)>>>(
      tk, tkr, p);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_lse_merge(const FcpbMergeArgs* a, void* stream) {
  if (!a) return fail(FCPB_ERR_INVALID, "null args");
  if (a->head_dim != 128) return fail(FCPB_ERR_UNSUPPORTED, "head_dim %d", a->head_dim);
  if (a->num_groups <= 0) return FCPB_OK;
  const int64_t rows = a->merged_tokens *   // one warp per (token, kMergeHeads heads)
                       ((a->num_q_heads + fcpb::aux::kMergeHeads - 1) / fcpb::aux::kMergeHeads);
  const int block = 256;
  const int64_t grid = (rows * 32 + block - 1) / block;
  fcpb::aux::lse_merge_kernel<<<static_cast<unsigned>(grid), block, 0,
                                static_cast<cudaStream_t>(stream)>>>(*a);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_bwd_preprocess(const void* o, const void* dout, const float* lse, float* lse2_t,
                        float* delta_t, int64_t t_pad, float* dq_accum, int64_t tokens,
                        int32_t num_q_heads, int32_t head_dim, void* stream) {
  if (head_dim != 128) return fail(FCPB_ERR_UNSUPPORTED, "head_dim %d", head_dim);
  if (t_pad < tokens || t_pad % 4) return fail(FCPB_ERR_INVALID, "bad t_pad %lld", (long long)t_pad);
  if (num_q_heads <= 0) return fail(FCPB_ERR_INVALID, "num_q_heads %d", num_q_heads);
  if (tokens == 0) return FCPB_OK;
  const int block = 256;
  const dim3 grid(static_cast<unsigned>((tokens + fcpb::aux::kPrepTokens - 1) / fcpb::aux::kPrepTokens),
                  static_cast<unsigned>((num_q_heads + fcpb::aux::kPrepMaxHeads - 1) / fcpb::aux::kPrepMaxHeads));
  fcpb::aux::bwd_preprocess_kernel<<<grid, block, 0,
                                     static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse, lse2_t,
      delta_t, t_pad, dq_accum, tokens, num_q_heads);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

// Exchange readiness flags, executed by the stream's front end (no SM): the persistent
// attention kernels fill every SM's shared memory, so a signalling *kernel* queued beside
// them waits for a whole launch before it can run.
namespace {
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValueFn stream_value_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<StreamValueFn>(p);
  return nullptr;
}
}  // namespace

int fcpb_stream_signal(void* flag, uint32_t value, void* stream) {
  static StreamValueFn fn = stream_value_fn("cuStreamWriteValue32");
  if (!fn) return fail(FCPB_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  if (!flag || reinterpret_cast<uintptr_t>(flag) % 4) return fail(FCPB_ERR_INVALID, "flag must be 4-byte aligned");
  // default flags: a stream-scoped system fence orders the stream's prior writes first
  const CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(FCPB_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  return FCPB_OK;
}

int fcpb_stream_wait(const void* flag, uint32_t value, void* stream) {
  static StreamValueFn fn = stream_value_fn("cuStreamWaitValue32");
  if (!fn) return fail(FCPB_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  if (!flag || reinterpret_cast<uintptr_t>(flag) % 4) return fail(FCPB_ERR_INVALID, "flag must be 4-byte aligned");
  // GEQ compares (int32)(*flag - value) >= 0: monotonically increasing epochs wrap safely
  const CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(FCPB_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return FCPB_OK;
}

int fcpb_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n <= 0) return FCPB_OK;
  if (n % 4) return fail(FCPB_ERR_INVALID, "n must be a multiple of 4");
  const int block = 256;
  const int64_t n4 = n / 4;
  int64_t grid = (n4 + block - 1) / block;
  if (grid > 148 * 16) grid = 148 * 16;
  fcpb::aux::f32_to_bf16_kernel<<<static_cast<unsigned>(grid), block, 0,
                                  static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<uint2*>(dst), n4);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_dkv_finalize(const float* local_k, const float* local_v, const float* staged_k,
                      const float* staged_v, const int32_t* row_ptr, const int32_t* src_rows,
                      int64_t n_rows, int64_t row_elems, void* out_k, void* out_v, void* stream) {
  if (n_rows <= 0) return FCPB_OK;
  if (row_elems % 4) return fail(FCPB_ERR_INVALID, "row_elems must be a multiple of 4");
  if (!local_k || !local_v || !row_ptr || !out_k || !out_v)
    return fail(FCPB_ERR_INVALID, "null local / row_ptr / output pointer");
  const int block = 256;
  const int64_t work = n_rows * (row_elems / 4);
  int64_t grid = (work + block - 1) / block;
  if (grid > 148 * 16) grid = 148 * 16;
  fcpb::aux::dkv_finalize_kernel<<<static_cast<unsigned>(grid), block, 0,
                                   static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(local_k), reinterpret_cast<const float4*>(local_v),
      reinterpret_cast<const float4*>(staged_k), reinterpret_cast<const float4*>(staged_v), row_ptr,
      src_rows, n_rows, row_elems / 4, reinterpret_cast<uint2*>(out_k), reinterpret_cast<uint2*>(out_v));
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_dkv_reduce(float* dst, const float* src, const int32_t* dst_rows, int64_t n_rows,
                    int64_t row_elems, void* stream) {
  if (n_rows <= 0) return FCPB_OK;
  if (row_elems % 4) return fail(FCPB_ERR_INVALID, "row_elems must be a multiple of 4");
  const int block = 256;
  const int64_t work = n_rows * (row_elems / 4);
  int64_t grid = (work + block - 1) / block;
  if (grid > 148 * 16) grid = 148 * 16;
  fcpb::aux::dkv_reduce_kernel<<<static_cast<unsigned>(grid), block, 0,
                                 static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), dst_rows, n_rows,
      row_elems / 4);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

// ---- peer-memory regions (K5/K6 transport): cudaMalloc + CUDA IPC handles.  Every call
// names its device explicitly and restores the caller's current device.
namespace {
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
static_assert(sizeof(FcpbIpcHandle) == sizeof(cudaIpcMemHandle_t), "IPC handle size");
}  // namespace

int fcpb_ipc_alloc(int device, size_t bytes, void** ptr, FcpbIpcHandle* handle) {
  if (!ptr || !handle || bytes == 0) return fail(FCPB_ERR_INVALID, "ipc_alloc: null pointer or zero size");
  DeviceGuard g(device);
  FCPB_CUDA(g.err);
  void* p = nullptr;
  FCPB_CUDA(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(FCPB_ERR_CUDA, "ipc_alloc: %s", cudaGetErrorString(e));
  }
  std::memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return FCPB_OK;
}

int fcpb_ipc_open(int device, const FcpbIpcHandle* handle, void** ptr) {
  if (!ptr || !handle) return fail(FCPB_ERR_INVALID, "ipc_open: null pointer");
  DeviceGuard g(device);
  FCPB_CUDA(g.err);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  FCPB_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return FCPB_OK;
}

int fcpb_ipc_close(int device, void* ptr) {
  DeviceGuard g(device);
  FCPB_CUDA(g.err);
  FCPB_CUDA(cudaIpcCloseMemHandle(ptr));
  return FCPB_OK;
}

int fcpb_ipc_free(int device, void* ptr) {
  DeviceGuard g(device);
  FCPB_CUDA(g.err);
  FCPB_CUDA(cudaFree(ptr));
  return FCPB_OK;
}

int fcpb_gather_copy(const void* segs, int32_t num_segs, int32_t num_ctas, void* stream) {
  if (num_segs < 0 || num_ctas <= 0) return fail(FCPB_ERR_INVALID, "gather_copy: bad counts");
  if (num_segs == 0) return FCPB_OK;
  if (!segs) return fail(FCPB_ERR_INVALID, "gather_copy: null segment table");
  const int grid = num_ctas < num_segs ? num_ctas : num_segs;
  fcpb::p2p::gather_kernel<<<grid, fcpb::p2p::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const fcpb::p2p::Seg*>(segs), num_segs);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int64_t fcpb_gather_seg_bytes(void) { return fcpb::p2p::kSegBytes; }

int fcpb_gather_copy_based(const void* segs, int32_t num_segs, const uint64_t* bases, int32_t num_bases,
                           int32_t num_ctas, void* stream) {
  static_assert(fcpb::p2p::kMaxBases == FCPB_GATHER_MAX_BASES, "header and kernel agree");
  if (num_segs < 0 || num_ctas <= 0 || num_bases < 0 || num_bases > fcpb::p2p::kMaxBases)
    return fail(FCPB_ERR_INVALID, "gather_copy_based: bad counts");
  if (num_segs == 0) return FCPB_OK;
  if (!segs || (num_bases && !bases)) return fail(FCPB_ERR_INVALID, "gather_copy_based: null table");
  fcpb::p2p::Bases b{};
  for (int i = 0; i < num_bases; ++i) b.p[i] = bases[i];
  const int grid = num_ctas < num_segs ? num_ctas : num_segs;
  fcpb::p2p::gather_based_kernel<<<grid, fcpb::p2p::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const fcpb::p2p::Seg*>(segs), num_segs, b);
  FCPB_CUDA(cudaGetLastError());
  return FCPB_OK;
}

int fcpb_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, void* stream) {
  if (width == 0 || height == 0) return FCPB_OK;
  if (!dst || !src) return fail(FCPB_ERR_INVALID, "copy_2d: null pointer");
  FCPB_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToDevice,
                              static_cast<cudaStream_t>(stream)));
  return FCPB_OK;
}

size_t fcpb_bwd_preprocess_bytes(int64_t tokens, int32_t num_q_heads) {
  const int64_t t_pad = (tokens + 3) / 4 * 4;
  return static_cast<size_t>(2) * num_q_heads * t_pad * sizeof(float);
}

size_t fcpb_fwd_partial_bytes(int64_t partial_rows, int32_t num_q_heads, int32_t head_dim) {
  return static_cast<size_t>(partial_rows) * num_q_heads * (static_cast<size_t>(head_dim) + 1) * sizeof(float);
}

size_t fcpb_ds_tile_bytes(int64_t ds_pairs, int32_t num_q_heads) {
  return static_cast<size_t>(ds_pairs) * num_q_heads * 128 * 128 * 2;
}

int fcpb_debug_counters(uint64_t* out, int n, int reset) {
  unsigned long long v = 0;
  FCPB_CUDA(cudaMemcpyFromSymbol(&v, fcpb::fwd::g_rescales, sizeof(v)));
  if (out && n > 0) out[0] = v;
  if (reset) {
    const unsigned long long z = 0;
    FCPB_CUDA(cudaMemcpyToSymbol(fcpb::fwd::g_rescales, &z, sizeof(z)));
  }
  return FCPB_OK;
}

#ifdef FCPB_TRACE
// Debug builds only (not part of include/fcpb.h): copy the bwd timeline of CTA 0.
__attribute__((visibility("default"))) int fcpb_debug_bwd_trace(unsigned long long* host, int n) {
  FCPB_CUDA(cudaMemcpyFromSymbol(host, fcpb::bwd::g_trace, sizeof(unsigned long long) * n));
  return FCPB_OK;
}
__attribute__((visibility("default"))) int fcpb_debug_dq_trace(unsigned long long* host, int n) {
  FCPB_CUDA(cudaMemcpyFromSymbol(host, fcpb::dq::g_trace, sizeof(unsigned long long) * n));
  return FCPB_OK;
}
__attribute__((visibility("default"))) int fcpb_debug_fwd_trace(unsigned long long* host, int n) {
  FCPB_CUDA(cudaMemcpyFromSymbol(host, fcpb::fwd::g_trace, sizeof(unsigned long long) * n));
  return FCPB_OK;
}
#endif

}  // extern "C"
