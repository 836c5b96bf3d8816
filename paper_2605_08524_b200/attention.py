"""Block-attention forward/backward entry points of one rank (K1-K4 launches).

``BlockAttention`` holds one rank's device work lists (built once per batch
from the ``ScheduleResult`` by ``worklist.build_rank_work``) and launches the
sm_100a kernels through the C ABI.  It is reused by every attention layer of
the batch.  The multi-GPU executor (``executor.py``) drives it wave by wave,
interleaved with the KV exchange; on one GPU ``forward``/``backward`` run the
whole rank at once.

Numerics: bf16 inputs, fp32 accumulation in TMEM, fp32 LSE (natural log);
dQ accumulates in TMEM over all KV and is written once in bf16; dK/dV are
fp32 (so received-chunk partials can be added at the owner) and rounded to bf16
at the end.
"""

from __future__ import annotations

import math

import torch

from . import native
from .costmodel import ModelConfig
from .errors import ParameterError
from .worklist import FwdWave, RankWork


def _dev_i32(arr, device):
    return torch.from_numpy(arr.copy()).to(device=device, dtype=torch.int32).contiguous()


def _check(t, name, shape, dtype=torch.bfloat16):
    if t is None:
        raise ParameterError(f"{name} is required")
    if not t.is_cuda:
        raise ParameterError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ParameterError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ParameterError(f"{name} shape {tuple(t.shape)} != expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ParameterError(f"{name} must be contiguous")


# per-rank tokens from which the head-major work order pays (see BlockAttention.__init__)
HEAD_MAJOR_MIN_TOKENS = 40960

class BlockAttention:
    def __init__(self, work: RankWork, cfg: ModelConfig, device=None,
                 softmax_scale: float | None = None, num_ctas: int = 0):
        if cfg.head_dim != 128:
            raise ParameterError("the sm_100a kernels are compiled for head_dim 128")
        self.lib = native.load()
        self.work = work
        self.cfg = cfg
        self.device = torch.device(device or "cuda")
        self.scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(cfg.head_dim)
        self.num_ctas = num_ctas
        lay = work.layout
        self.tokens = lay.tokens
        self.recv_tokens = lay.recv_tokens
        dev = self.device
        self._waves = [(w, _dev_i32(w.segments, dev), _dev_i32(w.kvrefs, dev), _dev_i32(w.items, dev))
                       for w in work.fwd.waves]
        f = work.fwd
        self._merge = None
        if len(f.merge_groups):
            self._merge = (_dev_i32(f.merge_groups, dev), _dev_i32(f.merge_part_rows, dev))
        self._bwd = [(b, _dev_i32(b.kvsegs, dev), _dev_i32(b.qrefs, dev), _dev_i32(b.items, dev))
                     for b in work.bwd]
        d = work.dq
        self._dq = (d, _dev_i32(d.segments, dev), _dev_i32(d.kvrefs, dev), _dev_i32(d.items, dev))
        self.launches = 0   # kernel launches issued by this object (bench accounting)
        props = torch.cuda.get_device_properties(self.device)
        self.sm_count = num_ctas or props.multi_processor_count
        # Materialised-dS backward: the dK/dV kernel writes every bf16 dS^T tile and dQ is a
        # grouped GEMM over them (attn_dqg_sm100.cuh) instead of recomputing S, dP and the
        # softmax.  Used when the tiles fit the budget (FCPB_DS=0/1 forces, FCPB_DS_BUDGET_GB).
        import os as _os
        ds_bytes = self.lib.fcpb_ds_tile_bytes(work.ds_pairs, cfg.q_heads)   # workspace query
        budget = float(_os.environ.get("FCPB_DS_BUDGET_GB", min(40.0, props.total_memory / 4 / 1e9))) * 1e9
        force = _os.environ.get("FCPB_DS")
        self.ds_mode = (force == "1") if force is not None else (0 < ds_bytes <= budget)
        self._ds = None
        self.ds_bytes = ds_bytes if self.ds_mode else 0
        if self.ds_mode:
            self._ds_pairs_base = [_dev_i32(b.pair_base, dev) for b in work.bwd]
            self._dq_pairs = (_dev_i32(work.dq.pair_ids, dev), _dev_i32(work.dq.pair_off, dev))
            self._ds_tiles = work.ds_pairs * cfg.q_heads
        import os
        # Work order of the dynamic scheduler.  Head-major (all items of one head, LPT order,
        # before the next head) keeps one head's Q/dO (or K/V) stream resident in L2: on C2
        # at N=1 it cut DRAM reads 17.8 -> 2.6 GB (dK/dV), 5.0 -> 1.4 GB (dQ), 3.5 -> 0.9 GB
        # (fwd) per launch, which under the 1 kW power cap is time.  But it starts the
        # largest items of the last heads late, a tail that grows as the per-rank work
        # shrinks.  Measured step time (profiles/r01_notes.md): head-major wins for C2 at N=1
        # (63K tokens/rank) and C3 at N=1/4 (>= 419K), head-interleaved wins for C2 at N=2/4
        # (31K / 16K tokens/rank) by 2.7% / 3.4%.  FCPB_SCHED="f,b,q" overrides.
        sched = os.environ.get("FCPB_SCHED", "")
        hm = 1 if self.tokens >= HEAD_MAJOR_MIN_TOKENS else 0
        flags = [int(x) for x in sched.split(",")] if sched else [hm, hm, hm]
        self.head_major = {"fwd": flags[0], "bwd": flags[1], "dq": flags[2]}
        # one dynamic-scheduler counter per kernel kind (zeroed by the C ABI before each launch)
        self._sched = torch.zeros(4, dtype=torch.int32, device=self.device)

    def _hm_lead(self, costs) -> int:
        """Head-major order: items that cannot fit one head's share of a CTA's work
        (cost > sum(costs) / #CTAs) still run heads-adjacent first, so no head's big item
        starts late.  C2 N=1 has a handful (about 0.8% faster than plain head-major).  On C3
        almost none; leading a fixed fifth there ran the bulk interleaved and cost 4.5%.
        FCPB_HM_LEAD=<n> overrides."""
        import os
        env = os.environ.get("FCPB_HM_LEAD")
        if env is not None:
            return int(env)
        if costs is None or len(costs) == 0:
            return 0
        return int((costs > costs.sum() / self.sm_count).sum())

    # ------------------------------------------------------------------ shapes
    def q_shape(self):
        return (self.tokens, self.cfg.q_heads, self.cfg.head_dim)

    def kv_shape(self, recv=False):
        return (self.recv_tokens if recv else self.tokens, self.cfg.kv_heads, self.cfg.head_dim)

    def _stream(self, stream):
        return native.stream_handle(stream if stream is not None else torch.cuda.current_stream())

    # ------------------------------------------------------------------ forward
    def alloc_forward_outputs(self):
        H, D = self.cfg.q_heads, self.cfg.head_dim
        o = torch.empty(self.q_shape(), dtype=torch.bfloat16, device=self.device)
        lse = torch.empty((self.tokens, H), dtype=torch.float32, device=self.device)
        rows = self.work.fwd.partial_rows
        op = lp = None
        if rows:
            op = torch.empty((rows, H, D), dtype=torch.float32, device=self.device)
            lp = torch.empty((rows, H), dtype=torch.float32, device=self.device)
        return o, lse, op, lp

    def forward_wave(self, idx, q, k, v, k_recv, v_recv, outs, stream=None):
        wave, segs, refs, items = self._waves[idx]
        o, lse, op, lp = outs
        a = native.FwdArgs()
        a.num_q_heads, a.num_kv_heads, a.head_dim = self.cfg.q_heads, self.cfg.kv_heads, self.cfg.head_dim
        a.softmax_scale = self.scale
        a.q, a.q_tokens = native.ptr(q), self.tokens
        a.k, a.v, a.kv_tokens = native.ptr(k), native.ptr(v), self.tokens
        a.k_recv, a.v_recv, a.kv_recv_tokens = native.ptr(k_recv), native.ptr(v_recv), self.recv_tokens
        a.o, a.lse = native.ptr(o), native.ptr(lse)
        a.o_partial, a.lse_partial = native.ptr(op), native.ptr(lp)
        a.partial_rows = self.work.fwd.partial_rows
        a.segments, a.num_segments = native.ptr(segs), len(wave.segments)
        a.kv_refs, a.num_kv_refs = native.ptr(refs), len(wave.kvrefs)
        a.items, a.num_items = native.ptr(items), len(wave.items)
        a.num_ctas = self.num_ctas
        a.head_major = self.head_major["fwd"]
        a.hm_lead = self._hm_lead(wave.costs)
        a.sched_counter = self._sched.data_ptr()
        native.check(self.lib.fcpb_attn_fwd(ctypes_ref(a), self._stream(stream)))
        self.launches += 1

    def merge(self, outs, stream=None):
        if self._merge is None:
            return
        o, lse, op, lp = outs
        groups, rows = self._merge
        a = native.MergeArgs()
        a.num_q_heads, a.head_dim = self.cfg.q_heads, self.cfg.head_dim
        a.o_partial, a.lse_partial = native.ptr(op), native.ptr(lp)
        a.groups, a.num_groups = native.ptr(groups), len(self.work.fwd.merge_groups)
        a.part_rows, a.merged_tokens = native.ptr(rows), self.work.fwd.merged_tokens
        a.o, a.lse = native.ptr(o), native.ptr(lse)
        native.check(self.lib.fcpb_lse_merge(ctypes_ref(a), self._stream(stream)))
        self.launches += 1

    @property
    def num_waves(self) -> int:
        return len(self._waves)

    def wave_stage(self, idx) -> int:
        return self._waves[idx][0].stage

    def forward(self, q, k, v, k_recv=None, v_recv=None, stream=None):
        """All waves then the merge; returns (o bf16 [T,Hq,D], lse fp32 [T,Hq])."""
        self.validate(q, k, v, k_recv, v_recv)
        outs = self.alloc_forward_outputs()
        for i in range(self.num_waves):
            self.forward_wave(i, q, k, v, k_recv, v_recv, outs, stream)
        self.merge(outs, stream)
        return outs[0], outs[1]

    def validate(self, q, k, v, k_recv=None, v_recv=None):
        _check(q, "q", self.q_shape())
        _check(k, "k", self.kv_shape())
        _check(v, "v", self.kv_shape())
        if self.recv_tokens:
            _check(k_recv, "k_recv", self.kv_shape(True))
            _check(v_recv, "v_recv", self.kv_shape(True))

    # ------------------------------------------------------------------ backward
    def backward_prepare(self, o, lse, do, stream=None):
        """-delta = -rowsum(dO*O) and -lse*log2(e), head-major [Hq, t_pad] fp32, for the
        dK/dV and dQ kernels.  Returns the (lse2_t, delta_t, t_pad) tuple they consume."""
        H = self.cfg.q_heads
        t_pad = (self.tokens + 3) // 4 * 4
        lse2_t = torch.empty((H, t_pad), dtype=torch.float32, device=self.device)
        delta_t = torch.empty((H, t_pad), dtype=torch.float32, device=self.device)
        native.check(self.lib.fcpb_bwd_preprocess(native.ptr(o), native.ptr(do), native.ptr(lse),
                                                  native.ptr(lse2_t), native.ptr(delta_t), t_pad,
                                                  None, self.tokens, H, self.cfg.head_dim,
                                                  self._stream(stream)))
        self.launches += 1
        return lse2_t, delta_t, t_pad

    def _ds_buffer(self):
        if self._ds is None:            # persistent across steps (one step's dS tiles)
            self._ds = torch.empty((self._ds_tiles, 128, 128), dtype=torch.bfloat16, device=self.device)
        return self._ds

    def backward_dq(self, q, k, v, k_recv, v_recv, prep, do, stream=None):
        """dQ of every local Q chunk -> bf16: a grouped GEMM over the dS tiles the dK/dV
        launches wrote (K2c, ds_mode), else the query-stationary recompute kernel (K2b)."""
        d, segs, refs, items = self._dq
        dq = torch.empty(self.q_shape(), dtype=torch.bfloat16, device=self.device)
        if self.ds_mode:
            a = native.DqDsArgs()
            a.num_q_heads, a.num_kv_heads, a.head_dim = self.cfg.q_heads, self.cfg.kv_heads, self.cfg.head_dim
            a.softmax_scale = self.scale
            a.ds, a.ds_tiles = native.ptr(self._ds_buffer()), self._ds_tiles
            a.k, a.kv_tokens = native.ptr(k), self.tokens
            a.k_recv, a.kv_recv_tokens = native.ptr(k_recv), self.recv_tokens
            a.dq = native.ptr(dq)
            a.segments, a.num_segments = native.ptr(segs), len(d.segments)
            a.kv_refs, a.num_kv_refs = native.ptr(refs), len(d.kvrefs)
            a.items, a.num_items = native.ptr(items), len(d.items)
            a.pair_ids, a.pair_off = native.ptr(self._dq_pairs[0]), native.ptr(self._dq_pairs[1])
            a.num_ctas = self.num_ctas
            a.head_major = self.head_major["dq"]
            a.hm_lead = self._hm_lead(d.costs)
            a.sched_counter = self._sched.data_ptr() + 8
            native.check(self.lib.fcpb_attn_bwd_dq_ds(ctypes_ref(a), self._stream(stream)))
            self.launches += 1
            return dq
        a = native.DqArgs()
        a.num_q_heads, a.num_kv_heads, a.head_dim = self.cfg.q_heads, self.cfg.kv_heads, self.cfg.head_dim
        a.softmax_scale = self.scale
        lse2_t, delta_t, t_pad = prep
        a.q, a.dout = native.ptr(q), native.ptr(do)
        a.lse2_t, a.delta_t, a.t_pad = native.ptr(lse2_t), native.ptr(delta_t), t_pad
        a.q_tokens = self.tokens
        a.k, a.v, a.kv_tokens = native.ptr(k), native.ptr(v), self.tokens
        a.k_recv, a.v_recv, a.kv_recv_tokens = native.ptr(k_recv), native.ptr(v_recv), self.recv_tokens
        a.dq = native.ptr(dq)
        a.segments, a.num_segments = native.ptr(segs), len(d.segments)
        a.kv_refs, a.num_kv_refs = native.ptr(refs), len(d.kvrefs)
        a.items, a.num_items = native.ptr(items), len(d.items)
        a.num_ctas = self.num_ctas
        a.head_major = self.head_major["dq"]
        a.hm_lead = self._hm_lead(d.costs)
        a.sched_counter = self._sched.data_ptr() + 8
        native.check(self.lib.fcpb_attn_bwd_dq(ctypes_ref(a), self._stream(stream)))
        self.launches += 1
        return dq

    def alloc_dkv(self, recv: bool):
        shape = self.kv_shape(recv)
        if shape[0] == 0:
            return None, None
        return (torch.empty(shape, dtype=torch.float32, device=self.device),
                torch.empty(shape, dtype=torch.float32, device=self.device))

    def backward_launch(self, recv: bool, q, k, v, k_recv, v_recv, prep, do,
                        dk, dv, dk_r, dv_r, stream=None, dk_out=None, dv_out=None):
        """K2 over the received (recv=True) or local chunks.  dk_out/dv_out (bf16): local
        chunks write their final dK/dV there directly -- only when no partials of this
        rank's chunks come back from peers."""
        for bi, (b, kvsegs, qrefs, items) in enumerate(self._bwd):
            if b.recv != recv:
                continue
            a = native.BwdArgs()
            a.num_q_heads, a.num_kv_heads, a.head_dim = self.cfg.q_heads, self.cfg.kv_heads, self.cfg.head_dim
            a.softmax_scale = self.scale
            lse2_t, delta_t, t_pad = prep
            a.q, a.dout = native.ptr(q), native.ptr(do)
            a.lse2_t, a.delta_t, a.t_pad = native.ptr(lse2_t), native.ptr(delta_t), t_pad
            a.q_tokens = self.tokens
            a.k, a.v, a.kv_tokens = native.ptr(k), native.ptr(v), self.tokens
            a.k_recv, a.v_recv, a.kv_recv_tokens = native.ptr(k_recv), native.ptr(v_recv), self.recv_tokens
            a.dq_accum, a.dk_accum, a.dv_accum = None, native.ptr(dk), native.ptr(dv)
            a.dk_recv_accum, a.dv_recv_accum = native.ptr(dk_r), native.ptr(dv_r)
            a.dk_out, a.dv_out = native.ptr(dk_out), native.ptr(dv_out)
            if self.ds_mode:
                a.ds_out = native.ptr(self._ds_buffer())
                a.pair_base = native.ptr(self._ds_pairs_base[bi])
            a.kvsegs, a.num_kvsegs = native.ptr(kvsegs), len(b.kvsegs)
            a.qrefs, a.num_qrefs = native.ptr(qrefs), len(b.qrefs)
            a.items, a.num_items = native.ptr(items), len(b.items)
            a.num_ctas = self.num_ctas
            a.head_major = self.head_major["bwd"]
            a.hm_lead = self._hm_lead(b.costs)
            a.sched_counter = self._sched.data_ptr() + 4
            native.check(self.lib.fcpb_attn_bwd(ctypes_ref(a), self._stream(stream)))
            self.launches += 1

    def to_bf16(self, src, stream=None):
        dst = torch.empty(src.shape, dtype=torch.bfloat16, device=self.device)
        native.check(self.lib.fcpb_f32_to_bf16(native.ptr(src), native.ptr(dst), src.numel(),
                                               self._stream(stream)))
        self.launches += 1
        return dst

    def reduce_dkv(self, dst, src, dst_rows, stream=None):
        """K4: dst[dst_rows[i]] += src[i] over token rows of Hkv*D floats."""
        row = self.cfg.kv_heads * self.cfg.head_dim
        native.check(self.lib.fcpb_dkv_reduce(native.ptr(dst), native.ptr(src), native.ptr(dst_rows),
                                              src.shape[0], row, self._stream(stream)))
        self.launches += 1

    def finalize_dkv(self, dk, dv, staged_k, staged_v, row_ptr, src_rows, stream=None):
        """K4 (fused): bf16(dK/dV local rows + their returned partials), one launch."""
        out_k = torch.empty(dk.shape, dtype=torch.bfloat16, device=self.device)
        out_v = torch.empty(dv.shape, dtype=torch.bfloat16, device=self.device)
        row = self.cfg.kv_heads * self.cfg.head_dim
        native.check(self.lib.fcpb_dkv_finalize(
            native.ptr(dk), native.ptr(dv), native.ptr(staged_k), native.ptr(staged_v),
            native.ptr(row_ptr), native.ptr(src_rows), dk.shape[0], row,
            native.ptr(out_k), native.ptr(out_v), self._stream(stream)))
        self.launches += 1
        return out_k, out_v

    def backward(self, q, k, v, o, lse, do, k_recv=None, v_recv=None, stream=None):
        """Single-rank backward.  Returns (dq, dk, dv) bf16 and, if the rank
        received KV, the fp32 (dk_recv, dv_recv) partials owed to their owners."""
        self.validate(q, k, v, k_recv, v_recv)
        _check(do, "do", self.q_shape())
        prep = self.backward_prepare(o, lse, do, stream)
        dk, dv = self.alloc_dkv(False)
        dk_r, dv_r = self.alloc_dkv(True)
        self.backward_launch(True, q, k, v, k_recv, v_recv, prep, do, dk, dv, dk_r, dv_r, stream)
        self.backward_launch(False, q, k, v, k_recv, v_recv, prep, do, dk, dv, dk_r, dv_r, stream)
        dq = self.backward_dq(q, k, v, k_recv, v_recv, prep, do, stream)
        return dq, self.to_bf16(dk, stream), self.to_bf16(dv, stream), dk_r, dv_r


def ctypes_ref(s):
    import ctypes
    return ctypes.byref(s)


class _FcpAttentionFn(torch.autograd.Function):
    """Autograd over one rank's block attention: a ``BlockAttention`` (single rank, no
    exchange) or an ``FcpExecutor`` (any N: the forward runs the K5 exchange and K3 merge,
    the backward the K6 return and K4).  Every rank must call it, in the same order, since
    the executor's exchange is collective."""

    @staticmethod
    def forward(ctx, q, k, v, runner):
        o, lse = runner.forward(q, k, v)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.runner = runner
        ctx.mark_non_differentiable(lse)
        return o, lse

    @staticmethod
    def backward(ctx, do, _dlse):
        q, k, v, o, lse = ctx.saved_tensors
        out = ctx.runner.backward(q, k, v, o, lse, do.contiguous())
        dq, dk, dv = out[:3]
        return dq, dk, dv, None


def fcp_attention(q, k, v, runner, return_lse: bool = False):
    """Differentiable FCP block attention of this rank's packed Q/K/V ([T, H, 128] bf16 in
    the plan's layout, ``worklist.rank_layout``).  ``runner``: an ``FcpExecutor`` (N >= 1,
    collective) or a ``BlockAttention`` (one rank without exchange).  Returns O (and the
    fp32 natural-log LSE when ``return_lse``)."""
    o, lse = _FcpAttentionFn.apply(q, k, v, runner)
    return (o, lse) if return_lse else o
