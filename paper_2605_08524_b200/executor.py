"""FCP executor: one rank's attention forward/backward with the KV exchange overlapped.

This is the GPU realisation of the reference's stage-synchronous model
(``simulator.py:154-232``):

forward   compute stream: wave -1 (local tiles, no dependency) is launched first;
          comm stream:    stage 0, 1, ... grouped P2P (NCCL) into the receive arena,
                          an event after each stage;
          compute stream: waits stage s's event, launches wave s (the tiles whose KV
                          arrived with stage s), ... then K3 merges the partials.
          All received KV stays resident (it is reused by the backward), so the
          transfer pipeline is never throttled by buffer reuse.
backward  compute: preprocess -> K2 dK/dV over *received* KV chunks (their partials
          are owed to the owners) -> event -> K2 dK/dV over local KV chunks ->
          K2b query-stationary dQ over all resident KV;
          comm:    after the event, every edge reversed: partials go back to the
          owners (K6), who add them with K4 once their local K2 finished.

Built once per batch from the ``ScheduleResult``; ``step`` can be called for
every layer.  One process per GPU (torchrun); ``group`` is the NCCL group.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import exchange
from .attention import BlockAttention
from .costmodel import ModelConfig
from .pipeline import ScheduleResult, plan_digest
from .worklist import LOCAL_WAVE, build_rank_work


class FcpExecutor:
    def __init__(self, result: ScheduleResult, rank: int, cfg: ModelConfig, device=None,
                 group=None, softmax_scale=None, num_ctas: int = 0, check_plan: bool = True):
        self.result = result
        self.rank = rank
        self.world = result.assignment.n_workers
        self.cfg = cfg
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.group = group
        if check_plan and self.world > 1:
            exchange.sync_plan_digest(plan_digest(result, cfg), group)
        self.work = build_rank_work(result, rank)
        self.layout = self.work.layout
        self.op = BlockAttention(self.work, cfg, self.device, softmax_scale, num_ctas)
        self.stages = exchange.build_stage_ops(result, self.layout)
        self.ret_rows, rounds, self.ret_tokens = exchange.return_staging_layout(self.stages)
        self.ret_rounds = [(torch.tensor(src, dtype=torch.int64, device=self.device),
                            torch.tensor(dst, dtype=torch.int32, device=self.device))
                           for src, dst in rounds]
        self.comm = torch.cuda.Stream(device=self.device, priority=-1)
        # wave index by stage
        self.wave_of_stage = {self.op.wave_stage(i): i for i in range(self.op.num_waves)}
        H, Hk, D = cfg.q_heads, cfg.kv_heads, cfg.head_dim
        R = self.layout.recv_tokens
        self.k_recv = torch.empty((R, Hk, D), dtype=torch.bfloat16, device=self.device) if R else None
        self.v_recv = torch.empty((R, Hk, D), dtype=torch.bfloat16, device=self.device) if R else None
        self.kv_bytes_per_token = 2 * Hk * D * 2

    # ------------------------------------------------------------------ accounting
    @property
    def tokens(self) -> int:
        return self.layout.tokens

    def flops(self) -> tuple[float, float]:
        """Algorithmic (fwd, bwd) FLOPs of this rank (reference costmodel.py:37-38, 26)."""
        fwd = self.work.pairs * self.cfg.flops_per_token_pair
        return fwd, fwd * self.cfg.backward_multiplier

    def exchange_bytes(self) -> dict:
        s, r = exchange.exchange_bytes(self.stages, self.kv_bytes_per_token)
        return {"fwd_send": s, "fwd_recv": r, "bwd_send": 2 * r, "bwd_recv": 2 * s}

    # ------------------------------------------------------------------ forward
    def forward(self, q, k, v):
        op = self.op
        cur = torch.cuda.current_stream(self.device)
        outs = op.alloc_forward_outputs()
        if LOCAL_WAVE in self.wave_of_stage:
            op.forward_wave(self.wave_of_stage[LOCAL_WAVE], q, k, v, self.k_recv, self.v_recv, outs, cur)
        if self.world > 1 and self.stages:
            self.comm.wait_stream(cur)       # k, v are ready
            events = []
            with torch.cuda.stream(self.comm):
                for st in self.stages:
                    if not st.empty:
                        exchange.wait_all(exchange.run_stage(st, (k, v), (self.k_recv, self.v_recv),
                                                             self.group))
                    ev = torch.cuda.Event()
                    ev.record(self.comm)
                    events.append(ev)
            for s, ev in enumerate(events):
                if s in self.wave_of_stage:
                    cur.wait_event(ev)
                    op.forward_wave(self.wave_of_stage[s], q, k, v, self.k_recv, self.v_recv, outs, cur)
            cur.wait_stream(self.comm)
        op.merge(outs, cur)
        return outs[0], outs[1]

    # ------------------------------------------------------------------ backward
    def backward(self, q, k, v, o, lse, do):
        op = self.op
        cur = torch.cuda.current_stream(self.device)
        prep = op.backward_prepare(o, lse, do, cur)
        dk, dv = op.alloc_dkv(False)
        dk_r, dv_r = op.alloc_dkv(True)
        args = (q, k, v, self.k_recv, self.v_recv, prep, do, dk, dv, dk_r, dv_r, cur)
        staged = None
        if self.world > 1 and self.stages:
            op.backward_launch(True, *args)
            self.comm.wait_stream(cur)
            Hk, D = self.cfg.kv_heads, self.cfg.head_dim
            with torch.cuda.stream(self.comm):
                sk = torch.empty((self.ret_tokens, Hk, D), dtype=torch.float32, device=self.device)
                sv = torch.empty_like(sk)
                exchange.wait_all(exchange.run_return(self.stages, (dk_r, dv_r), (sk, sv),
                                                      self.ret_rows, self.group))
            staged = (sk, sv)
        op.backward_launch(False, *args)
        dq = op.backward_dq(q, k, v, self.k_recv, self.v_recv, prep, do, cur)
        if staged is not None:
            cur.wait_stream(self.comm)
            for src, dst in self.ret_rounds:        # K4, one race-free round per receiver rank
                op.reduce_dkv(dk, staged[0].index_select(0, src), dst, cur)
                op.reduce_dkv(dv, staged[1].index_select(0, src), dst, cur)
        return dq, op.to_bf16(dk, cur), op.to_bf16(dv, cur)

    def step(self, q, k, v, do):
        """One attention layer fwd+bwd; returns (o, lse, dq, dk, dv)."""
        o, lse = self.forward(q, k, v)
        dq, dk, dv = self.backward(q, k, v, o, lse, do)
        return o, lse, dq, dk, dv
