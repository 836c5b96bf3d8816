"""FCP executor: one rank's attention forward/backward with the KV exchange overlapped.

This is the GPU realisation of the reference's stage-synchronous model
(``simulator.py:154-232``):

forward   compute stream: wave -1 (local tiles, no dependency) is launched first;
          comm stream:    stage 0, 1, ... copy-engine pulls into the receive arena,
                          an event after each stage;
          compute stream: waits stage s's event, launches wave s (the tiles whose KV
                          arrived with stage s), ... then K3 merges the partials.
          All received KV stays resident (it is reused by the backward), so the
          transfer pipeline is never throttled by buffer reuse.
backward  compute: preprocess -> K2 dK/dV over *received* KV chunks (partials land in
          symmetric memory) -> K2 dK/dV over local KV chunks -> K2b dQ over all resident KV;
          comm:    barrier, then every owner pulls the partials of its chunks back along
          the reversed plan edges (K6) while the local kernels run; K4 adds them.
Transport: copy-engine pulls from IPC-mapped peer memory (``p2p.py``) -- no SMs taken
from the persistent kernels; measured ~5x faster than NCCL send/recv here.

Built once per batch from the ``ScheduleResult``; ``step`` can be called for
every layer.  One process per GPU (torchrun); ``group`` is the NCCL group.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import exchange
from .attention import BlockAttention
from .costmodel import ModelConfig
from .pipeline import ScheduleResult, plan_digest
from .worklist import LOCAL_WAVE, PRE_WAVE, build_rank_work


def kernel_config(cfg: ModelConfig):
    """(config the sm_100a kernels run, q-head replication) for a user config.  The kernels
    are compiled for head_dim 128 and an even GQA group (a forward CTA serves two q-heads of
    one K/V head).  Smaller head dims run zero-padded to 128 (the scores, P, O and every
    gradient are unchanged, the padded columns stay zero), and an odd group runs every q-head
    twice with a zero dO for the copy (its dS, hence its dK/dV contribution, is exactly zero);
    the softmax scale stays 1/sqrt(user head_dim).  Exact, at up to 4x the tensor work of a
    native kernel -- this serves the tiny C1 model (Hq = Hkv = 4, D = 64)."""
    from .errors import ParameterError
    if cfg.head_dim > 128 or cfg.head_dim % 8:
        raise ParameterError(f"head_dim {cfg.head_dim}: the kernels support multiples of 8 up to 128")
    if cfg.kv_heads <= 0 or cfg.q_heads % cfg.kv_heads:
        raise ParameterError(f"q_heads {cfg.q_heads} is not a multiple of kv_heads {cfg.kv_heads}")
    rep = 1 if (cfg.q_heads // cfg.kv_heads) % 2 == 0 else 2
    if rep == 1 and cfg.head_dim == 128:
        return cfg, 1
    return ModelConfig(q_heads=cfg.q_heads * rep, kv_heads=cfg.kv_heads, head_dim=128,
                       dtype_bytes=cfg.dtype_bytes), rep


def pad_head_dim(x, d_to: int = 128):
    """[..., D] -> [..., 128], zero-padded (kernel_config)."""
    d = x.shape[-1]
    return x if d == d_to else torch.nn.functional.pad(x, (0, d_to - d)).contiguous()


def replicate_q_heads(x, rep: int, zero_copy: bool = False):
    """[T, Hq, ...] -> [T, rep*Hq, ...]: every q-head twice, interleaved (heads 2h and 2h+1
    map to h's K/V head under the doubled group); the copy is zero when zero_copy (the dO and
    O of the duplicates, whose dS and gradients then vanish exactly)."""
    if rep == 1:
        return x
    if zero_copy:
        return torch.stack([x, torch.zeros_like(x)], dim=2).flatten(1, 2).contiguous()
    return x.repeat_interleave(rep, dim=1).contiguous()


def unreplicate_q(x, rep: int, d: int):
    """Kernel-shaped Q-side output ([T, rep*Hq, 128] or [T, rep*Hq]) -> user shape."""
    if rep > 1:
        x = x[:, 0::rep]
    if x.dim() == 3 and x.shape[-1] != d:
        x = x[..., :d]
    return x.contiguous()


class FcpExecutor:
    def __init__(self, result: ScheduleResult, rank: int, cfg: ModelConfig, device=None,
                 group=None, softmax_scale=None, num_ctas: int = 0, check_plan: bool = True,
                 comm_sms: int | None = None, resident=None):
        self.result = result
        self.rank = rank
        self.world = result.assignment.n_workers
        self.user_cfg = cfg
        # the kernels' shapes (kernel_config): D padded to 128, q-heads doubled for odd groups
        kcfg, self.q_rep = kernel_config(cfg)
        self.adapt = kcfg is not cfg
        if self.adapt and softmax_scale is None:
            import math
            softmax_scale = 1.0 / math.sqrt(cfg.head_dim)
        self.cfg = cfg = kcfg
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.group = group
        if check_plan and self.world > 1:
            exchange.sync_plan_digest(plan_digest(result, self.user_cfg), group)
        # resident: chunks whose rows are in place before a reshuffle into the FCP layout
        # completes (Reshuffler.resident_chunks); their local tiles form PRE_WAVE
        self.resident = frozenset(resident or ())
        self.work = build_rank_work(result, rank, resident=self.resident)
        self.fuse_remote = self._fuse_remote_waves(result, rank, cfg)
        if self.fuse_remote:
            self.work = build_rank_work(result, rank, fuse_remote=self.fuse_remote, resident=self.resident)
        self.layout = self.work.layout
        self.op = BlockAttention(self.work, cfg, self.device, softmax_scale, num_ctas)
        # The exchange runs on copy engines (p2p.SymmetricExchange), so the persistent
        # kernels keep every SM; comm_sms > 0 would shrink their grids while pulls run.
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        self.overlap_ctas = max(1, sms - comm_sms) if (self.world > 1 and comm_sms) else 0
        self.stages = exchange.build_stage_ops(result, self.layout)
        from .distributor import chunk_placement
        from .worklist import rank_layout
        layouts = [self.layout if r == rank else rank_layout(result, r) for r in range(self.world)]
        # K6: partials of my chunks come back from every rank that consumed them
        self.returns = exchange.owner_returns(layouts, chunk_placement(result.assignment, result.units),
                                              rank)
        self.ret_rows, rounds, self.ret_tokens = exchange.return_staging_layout(self.returns)
        # K4 (fused finalize): per local row, the staging rows of its returned partials (CSR)
        import numpy as np
        T = self.layout.tokens
        dst_all = np.array([d for _, dst in rounds for d in dst], dtype=np.int64)
        src_all = np.array([x for src, _ in rounds for x in src], dtype=np.int64)
        order = np.argsort(dst_all, kind="stable")
        row_ptr = np.zeros(T + 1, dtype=np.int32)
        if len(dst_all):
            row_ptr[1:] = np.cumsum(np.bincount(dst_all, minlength=T))
        self.ret_row_ptr = torch.tensor(row_ptr, dtype=torch.int32, device=self.device)
        self.ret_src_rows = torch.tensor(src_all[order] if len(src_all) else np.zeros(1, np.int64),
                                         dtype=torch.int32, device=self.device)
        self.comm = torch.cuda.Stream(device=self.device, priority=-1)
        self.xchg = None
        if self.world > 1:
            from .p2p import SymmetricExchange
            self.xchg = SymmetricExchange(result, rank, cfg, self.device, group)
        # wave index by stage
        self.wave_of_stage = {self.op.wave_stage(i): i for i in range(self.op.num_waves)}
        # One forward wave after the exchange (fuse_remote="all"): nothing overlaps the pulls,
        # so they run as the K5 pull kernel on every SM instead of on copy engines
        # (FCPB_PULL=ce keeps the copy engines).
        self.sm_pull = (self.xchg is not None and self.fuse_remote == "all"
                        and LOCAL_WAVE not in self.wave_of_stage
                        and os.environ.get("FCPB_PULL", "sm") == "sm")
        H, Hk, D = cfg.q_heads, cfg.kv_heads, cfg.head_dim
        R = self.layout.recv_tokens
        # receive arena: K plane then V plane, so one 2-D copy moves a run of both
        self.kv_recv = torch.empty((2, R, Hk, D), dtype=torch.bfloat16, device=self.device) if R else None
        self.k_recv = self.kv_recv[0] if R else None
        self.v_recv = self.kv_recv[1] if R else None
        self.kv_bytes_per_token = 2 * Hk * D * 2
        self._marks = None          # optional per-phase CUDA-event timeline (see timeline())
        self._rs_stream = None      # forward_user: the reshuffle's remote pulls

    def _fuse_remote_waves(self, result, rank, cfg):
        """How the forward groups a rank's tiles into waves.  With the copy-engine exchange
        (550-700 GB/s per rank at N=2, 2-D pulls of merged runs) a rank's pulls are short
        next to its compute, so by default every tile goes into ONE wave released by the
        last arrival stage ("all"): no fp32 partials, no LSE merge and one launch tail, for
        the price of the exposed exchange.  Measured at N=4 (`gpurun_out/abm1_*`): C2 4.78 vs
        4.80-4.88 ms, C3 621.4-621.7 vs 621.9-623.6 ms against a local wave overlapped with
        the pulls plus one fused remote wave.  FCPB_FUSE_REMOTE=0/1/all/resume overrides."""
        env = os.environ.get("FCPB_FUSE_REMOTE")
        if env is not None:
            return env if env in ("all", "resume") else env == "1"
        waves = self.work.fwd.waves
        if self.world == 1 or not any(w.stage >= 0 for w in waves):
            return False
        return "all"

    def kv_input_buffers(self):
        """(k, v) [T, Hkv, D] bf16 buffers to write this rank's K/V into before ``forward``.
        At N > 1 they are the K/V planes of the exchange region, so the peers read them in
        place and the step skips the publish copy; at N = 1 plain tensors.  Writes issued on
        the current stream after this call are ordered after the peers' pulls of the previous
        step (the comm stream ends each forward with the "K/V consumed" barrier)."""
        if self.xchg is not None and not self.adapt:
            torch.cuda.current_stream(self.device).wait_stream(self.comm)
            return self.xchg.kv_views()
        shape = (self.layout.tokens, self.user_cfg.kv_heads, self.user_cfg.head_dim)
        return (torch.empty(shape, dtype=torch.bfloat16, device=self.device),
                torch.empty(shape, dtype=torch.bfloat16, device=self.device))

    # ------------------------------------------------------------------ timeline
    def timeline(self, enabled: bool = True):
        """Record CUDA events at phase boundaries of the next steps (compute and comm
        streams); ``phases()`` returns the measured milliseconds per phase."""
        self._marks = [] if enabled else None

    def _mark(self, name, stream):
        if self._marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            self._marks.append((name, ev))

    def phases(self) -> dict:
        """Average ms from the step's first mark to every later mark (compute and comm
        stream marks interleaved), keyed '<order>:<name>'."""
        if not self._marks:
            return {}
        torch.cuda.synchronize(self.device)
        out: dict = {}
        steps, t0, k = 0, None, 0
        for name, ev in self._marks:
            if name == "step_begin":
                t0, k, steps = ev, 0, steps + 1
                continue
            k += 1
            key = f"{k:02d}:{name}"
            out[key] = out.get(key, 0.0) + t0.elapsed_time(ev)
        return {kk: v / max(steps, 1) for kk, v in out.items()}

    # ------------------------------------------------------------------ accounting
    @property
    def tokens(self) -> int:
        return self.layout.tokens

    def flops(self) -> tuple[float, float]:
        """Algorithmic (fwd, bwd) FLOPs of this rank (reference costmodel.py:37-38, 26)."""
        fwd = self.work.pairs * self.user_cfg.flops_per_token_pair
        return fwd, fwd * self.user_cfg.backward_multiplier

    def exchange_bytes(self) -> dict:
        s, r = exchange.exchange_bytes(self.stages, self.kv_bytes_per_token)
        return {"fwd_send": s, "fwd_recv": r, "bwd_send": 2 * r, "bwd_recv": 2 * s}

    # ------------------------------------------------------------------ forward
    # ------------------------------------------------------------------ shape adapter
    def _pad_d(self, x):
        return pad_head_dim(x)

    def _q_in(self, x, zero_copy=False):
        return replicate_q_heads(pad_head_dim(x), self.q_rep, zero_copy)

    def _q_out(self, x):
        return unreplicate_q(x, self.q_rep, self.user_cfg.head_dim)

    def forward(self, q, k, v, pre_event=None):
        """O, LSE of this rank's Q rows.  pre_event: the inputs are complete only once this
        event has fired (a reshuffle still in flight, ``forward_user``); the PRE_WAVE tiles,
        whose rows were in place before, run first, then the stream waits for it.  A callable
        pre_event is called right after the PRE_WAVE launch and returns the event."""
        if self.adapt:
            if pre_event is not None:
                if callable(pre_event):
                    pre_event = pre_event()
                torch.cuda.current_stream(self.device).wait_event(pre_event)
            o, lse = self._forward(self._q_in(q), self._pad_d(k), self._pad_d(v))
            return self._q_out(o), self._q_out(lse)
        return self._forward(q, k, v, pre_event)

    def _forward(self, q, k, v, pre_event=None):
        op = self.op
        cur = torch.cuda.current_stream(self.device)
        outs = op.alloc_forward_outputs()
        self._mark("step_begin", cur)
        if PRE_WAVE in self.wave_of_stage:
            op.forward_wave(self.wave_of_stage[PRE_WAVE], q, k, v, self.k_recv, self.v_recv, outs, cur)
            self._mark("fwd_pre", cur)
        if pre_event is not None:
            if callable(pre_event):      # a deferred reshuffle: enqueue it behind the PRE_WAVE
                pre_event = pre_event()
            cur.wait_event(pre_event)
        x = self.xchg
        events = []
        if x is not None and self.stages and self.sm_pull:
            cur.wait_stream(self.comm)
            x.publish_kv(k, v)
            x.barrier("kv", 0)                          # (compute stream) everyone's K/V readable
            x.gather_all(self.kv_recv, cur)             # every stage's pulls, one launch
            self._mark("comm_stage_done", cur)
            events = [None] * len(self.stages)
            self.comm.wait_stream(cur)
            with torch.cuda.stream(self.comm):
                x.barrier("kv", 1)                      # all pulls done: K/V reusable
        elif x is not None and self.stages:
            # previous step's pulls of our K/V are complete (comm-stream order + barrier)
            cur.wait_stream(self.comm)
            x.publish_kv(k, v)
            self.comm.wait_stream(cur)
            with torch.cuda.stream(self.comm):
                x.barrier("kv", 0)                      # everyone's K/V readable
                for s_idx in range(len(self.stages)):
                    x.pull_stage(s_idx, self.kv_recv)
                    ev = torch.cuda.Event()
                    ev.record(self.comm)
                    events.append(ev)
                    self._mark("comm_stage_done", self.comm)
                x.barrier("kv", 1)                      # all pulls done: K/V reusable
        if LOCAL_WAVE in self.wave_of_stage:
            op.forward_wave(self.wave_of_stage[LOCAL_WAVE], q, k, v, self.k_recv, self.v_recv, outs, cur)
            self._mark("fwd_local", cur)
        for s_idx, ev in enumerate(events):
            if s_idx in self.wave_of_stage:
                if ev is not None:
                    cur.wait_event(ev)
                op.forward_wave(self.wave_of_stage[s_idx], q, k, v, self.k_recv, self.v_recv, outs, cur)
                self._mark(f"fwd_wave{s_idx}", cur)
        if events:
            self._mark("fwd_remote", cur)
        op.merge(outs, cur)
        self._mark("fwd_merge", cur)
        return outs[0], outs[1]

    # ------------------------------------------------------------------ backward
    def backward(self, q, k, v, o, lse, do):
        if self.adapt:
            lse_k = lse.repeat_interleave(self.q_rep, dim=1).contiguous() if self.q_rep > 1 else lse
            dq, dk, dv = self._backward(self._q_in(q), self._pad_d(k), self._pad_d(v),
                                        self._q_in(o, zero_copy=True), lse_k, self._q_in(do, zero_copy=True))
            D = self.user_cfg.head_dim
            return self._q_out(dq), dk[..., :D].contiguous(), dv[..., :D].contiguous()
        return self._backward(q, k, v, o, lse, do)

    def _backward(self, q, k, v, o, lse, do):
        op = self.op
        cur = torch.cuda.current_stream(self.device)
        prep = op.backward_prepare(o, lse, do, cur)
        self._mark("bwd_prep", cur)
        final = self.ret_tokens == 0     # see below: dK/dV written straight to bf16
        dk, dv = (None, None) if final else op.alloc_dkv(False)
        x = self.xchg
        staged = None
        if x is not None and self.stages:
            dk_r, dv_r = x.partial_views()              # partials land in symmetric memory
            args = (q, k, v, self.k_recv, self.v_recv, prep, do, dk, dv, dk_r, dv_r, cur)
            op.backward_launch(True, *args)
            self._mark("bwd_dkv_recv", cur)
            Hk, D = self.cfg.kv_heads, self.cfg.head_dim
            staging = torch.empty((2, self.ret_tokens, Hk, D), dtype=torch.float32, device=self.device)
            sk, sv = staging[0], staging[1]
            self.comm.wait_stream(cur)
            with torch.cuda.stream(self.comm):
                if x.BARRIER == "kernel":
                    x.barrier("part", 0)                # every rank's partials written
                    x.pull_returns(self.returns, staging, self.ret_rows)
                else:
                    # my partials are written; each owner pulls a consumer's partials as
                    # soon as that consumer has signalled (no wait for the slowest rank)
                    x.signal_all("part", 0)
                    x.pull_returns(self.returns, staging, self.ret_rows, per_peer_ready=True)
                x.barrier("part", 1)                    # pulled: partial buffers reusable
                self._mark("comm_return_done", self.comm)
            staged = (sk, sv)
        else:
            dk_r, dv_r = op.alloc_dkv(True)
            args = (q, k, v, self.k_recv, self.v_recv, prep, do, dk, dv, dk_r, dv_r, cur)
        # No partial of this rank's chunks comes back (always at N=1): the dK/dV kernel
        # writes the final bf16 gradients itself (no fp32 round trip, no convert launches).
        if final:
            dk_b = torch.empty(k.shape, dtype=torch.bfloat16, device=self.device)
            dv_b = torch.empty(v.shape, dtype=torch.bfloat16, device=self.device)
            op.backward_launch(False, *args, dk_out=dk_b, dv_out=dv_b)
        else:
            op.backward_launch(False, *args)
        self._mark("bwd_dkv_local", cur)
        dq = op.backward_dq(q, k, v, self.k_recv, self.v_recv, prep, do, cur)
        self._mark("bwd_dq", cur)
        if staged is not None:
            # the comm stream's return pulls and barriers order the reuse of the partial
            # buffers, even on a rank none of whose chunks was consumed remotely
            cur.wait_stream(self.comm)
            self._mark("bwd_wait_return", cur)
            if not final:
                # K4: local rows + every returned partial, rounded once to bf16 (one launch)
                dk_b, dv_b = op.finalize_dkv(dk, dv, staged[0], staged[1], self.ret_row_ptr,
                                             self.ret_src_rows, cur)
                final = True
        out = (dq, dk_b, dv_b) if final else (dq, op.to_bf16(dk, cur), op.to_bf16(dv, cur))
        self._mark("bwd_reduce_convert", cur)
        return out

    def exchange_benchmark(self, reps: int = 5) -> dict | None:
        """Isolated exchange bandwidth of this rank (no attention running), over the
        transport the step uses (the K5 pull kernel when ``sm_pull``, else copy engines):
        the forward K/V pulls of every stage and the backward partial-dKV returns, each
        bracketed by the same symmetric-memory barriers the step uses and timed with CUDA
        events on the comm stream.  GB/s = bytes this rank receives / time (the read
        direction of its NVLink ports; B200 NVLink 5: 900 GB/s per direction)."""
        x = self.xchg
        if x is None or not self.stages:
            return None
        Hk, D = self.cfg.kv_heads, self.cfg.head_dim
        staging = torch.empty((2, max(self.ret_tokens, 1), Hk, D), dtype=torch.float32, device=self.device)
        b = self.exchange_bytes()
        out = {}
        for name, nbytes in (("fwd_kv_pull", b["fwd_recv"]), ("bwd_dkv_return", b["bwd_recv"])):
            times = []
            for _ in range(reps + 1):
                torch.cuda.synchronize(self.device)
                s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(self.comm):
                    which = "kv" if name == "fwd_kv_pull" else "part"
                    x.barrier(which, 0)
                    s0.record(self.comm)
                    if which == "kv" and self.sm_pull:
                        x.gather_all(self.kv_recv, self.comm)
                    elif which == "kv":
                        for s_idx in range(len(self.stages)):
                            x.pull_stage(s_idx, self.kv_recv)
                    else:
                        x.pull_returns(self.returns, staging, self.ret_rows)
                    e0.record(self.comm)
                    x.barrier(which, 1)
                torch.cuda.synchronize(self.device)
                times.append(s0.elapsed_time(e0))
            t = sorted(times[1:])[len(times[1:]) // 2]
            out[name] = {"bytes": nbytes, "ms": t, "GBps": nbytes / (t * 1e-3) / 1e9 if t > 0 else None}
        out["peak_GBps_per_direction"] = 900.0
        return out

    def measured_report(self, q, k, v, do, reps: int = 3):
        """A measured counterpart of the reference's analytic ``simulate()`` report
        (``simulator.py:60-70`` / ``simmodel.SimReport``) for one fwd+bwd step:

        * ``total_time``: device step time in seconds (max over ranks);
        * ``per_worker[r]``: compute_time = summed durations of rank r's attention launches
          (CUDA events around each), send/recv_time = its exchange bytes over the isolated
          copy-engine pull time, idle_time = total - compute, eta = total / compute;
        * ``stages``: one record per coalesced stage, the isolated pull time of this rank;
        * ``total_flops``: the reference accounting, 3.5 * 4*Hq*D * visible pairs of the batch;
        * ``total_bytes``: the plan's edge bytes (``planner.py:81-102``).
        Collective over the process group when world > 1."""
        import torch.distributed as dist
        from .distributor import worker_loads
        from .simmodel import SimReport, StageRecord, WorkerStats
        op = self.op
        cur = torch.cuda.current_stream(self.device)
        spans = []
        names = ("forward_wave", "merge", "backward_prepare", "backward_launch", "backward_dq",
                 "reduce_dkv", "finalize_dkv", "to_bf16")
        orig = {n: getattr(op, n) for n in names}

        def wrap(fn):
            def w(*a, **kw):
                s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(cur)
                out = fn(*a, **kw)
                e0.record(cur)
                spans.append((s0, e0))
                return out
            return w

        self.step(q, k, v, do)                          # warm
        torch.cuda.synchronize(self.device)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(cur)
        for _ in range(reps):
            self.step(q, k, v, do)
        t1.record(cur)
        torch.cuda.synchronize(self.device)
        total = t0.elapsed_time(t1) / reps / 1e3
        for n in names:
            setattr(op, n, wrap(orig[n]))
        try:
            for _ in range(reps):
                self.step(q, k, v, do)
            torch.cuda.synchronize(self.device)
        finally:
            for n in names:
                setattr(op, n, orig[n])
        compute = sum(a.elapsed_time(b) for a, b in spans) / reps / 1e3
        xb = self.exchange_benchmark(reps) if self.world > 1 else None
        b = self.exchange_bytes()
        send = recv = 0.0
        if xb:
            rate = xb["fwd_kv_pull"]["bytes"] / max(xb["fwd_kv_pull"]["ms"] * 1e-3, 1e-12)
            if rate > 0:                # a rank that receives nothing has no pull rate
                send, recv = b["fwd_send"] / rate, b["fwd_recv"] / rate
        stages = []
        if self.xchg is not None and self.stages:
            for s_idx in range(len(self.stages)):
                torch.cuda.synchronize(self.device)
                s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(self.comm):
                    self.xchg.barrier("kv", 0)
                    s0.record(self.comm)
                    self.xchg.pull_stage(s_idx, self.kv_recv)
                    e0.record(self.comm)
                    self.xchg.barrier("kv", 1)
                torch.cuda.synchronize(self.device)
                stages.append(StageRecord(s0.elapsed_time(e0) / 1e3, "comm"))
        mine = (total, compute, send, recv)
        if self.world > 1 and dist.is_initialized():
            allv = [None] * self.world
            dist.all_gather_object(allv, mine, group=self.group)
        else:
            allv = [mine]
        t_max = max(x[0] for x in allv)
        per = [WorkerStats(compute_time=c, send_time=sd, recv_time=rv, idle_time=t_max - c,
                           eta=t_max / c if c > 0 else 1.0) for _, c, sd, rv in allv]
        loads = worker_loads(self.result.assignment, self.result.units, self.result.deps, self.user_cfg)
        flops = 3.5 * float(sum(loads.compute_flops))      # distributor.py:151-155 accounting
        nbytes = int(sum(e.nbytes for st in self.result.plan.stages for e in st))
        return SimReport(t_max, per, stages, flops, nbytes)

    def close(self) -> None:
        """Release the peer-memory regions of this batch's exchange (collective at N > 1:
        every rank calls it, after its last step; the executor is unusable afterwards)."""
        if self.xchg is not None:
            torch.cuda.synchronize(self.device)
            self.xchg.close()
            self.xchg = None

    def forward_user(self, rs, q_u, k_u, v_u, overlap: bool | None = None):
        """Forward from the user's layout.  K/V land directly
        in ``kv_input_buffers`` (no publish copy at N > 1).  Returns the FCP-layout (q, k, v)
        and (o, lse).

        overlap=True (default; FCPB_RESHUFFLE_OVERLAP=0 flips it): the reshuffler copies the
        rows that stay on this rank (one gather launch), the PRE_WAVE tiles (rows in place;
        build the executor with ``resident=rs.resident_chunks()``) are enqueued next, and the
        remote pulls run on copy engines on a side stream beside them.  overlap=False: the
        whole to-FCP move first (remote pulls as the K5 pull kernel), then the forward.  C2 at
        N=2 (scripts/forward_user_probe.py): 2.32 vs 2.58 ms.
        """
        if overlap is None:
            overlap = os.environ.get("FCPB_RESHUFFLE_OVERLAP", "1") == "1"
        H, D = self.user_cfg.q_heads, self.user_cfg.head_dim
        q = torch.empty((self.layout.tokens, H, D), dtype=q_u.dtype, device=self.device)
        k, v = self.kv_input_buffers()
        if not overlap:
            q, k, v = rs._move([q_u, k_u, v_u], rs.plan.to_fcp, rs.plan.user_tokens, rs.plan.fcp_tokens,
                               outs=[q, k, v])
            return (q, k, v), self.forward(q, k, v)
        if self._rs_stream is None:
            self._rs_stream = torch.cuda.Stream(device=self.device)
        (q, k, v), start = rs._move([q_u, k_u, v_u], rs.plan.to_fcp, rs.plan.user_tokens,
                                    rs.plan.fcp_tokens, outs=[q, k, v], remote_stream=self._rs_stream,
                                    defer_remote=True)
        o, lse = self.forward(q, k, v, pre_event=start)
        return (q, k, v), (o, lse)

    def attention(self, q, k, v, return_lse: bool = False):
        """Differentiable attention through this executor (``attention.fcp_attention``):
        ``loss.backward()`` runs ``backward`` -- the dK/dV return included -- on every rank."""
        from .attention import fcp_attention
        return fcp_attention(q, k, v, self, return_lse)

    def step(self, q, k, v, do):
        """One attention layer fwd+bwd; returns (o, lse, dq, dk, dv)."""
        o, lse = self.forward(q, k, v)
        dq, dk, dv = self.backward(q, k, v, o, lse, do)
        return o, lse, dq, dk, dv
