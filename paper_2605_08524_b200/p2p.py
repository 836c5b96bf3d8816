"""K5/K6 transport: copy-engine pulls from symmetric (IPC-mapped) peer memory over NVLink.

Measured on the B200 box: NCCL grouped send/recv moved the FCP stages at ~45 GB/s
(2 MB messages, and its kernels compete with the persistent attention kernels for
SMs), while ``cudaMemcpyAsync`` pulls from a peer's mapped buffer reach ~250 GB/s
per direction for the same 2 MB chunks with *no* SM use.  Per the north star
("NCCL grouped send/recv, or in-kernel P2P, whichever measures faster") the executor
uses the pulls; ``exchange.run_stage`` (torch.distributed P2P) stays as the
transport-agnostic reference of the same plan that the gloo CPU tests exercise.

Buffers (torch symmetric memory, same size on every rank):

* ``kv``   bf16 [2, T_max, Hkv, D] -- each rank's own K and V (copied in at step start)
* ``part`` fp32 [2, R_max, Hkv, D] -- dK/dV partials of the chunks a rank *received*
  (written directly by the dK/dV kernel), pulled back by the chunk owners.

* ``flags`` int32 [4, world] -- readiness words written by the peers' streams.

Ordering: an all-rank barrier after the K/V copy (everyone's K/V is readable), after
the forward pulls (K/V may be overwritten next step), after the partials are written,
and after the return pulls.  The barrier is stream memory operations on the flag words
(``fcpb_stream_signal`` / ``fcpb_stream_wait``), executed without an SM.  Each plan edge (reference
``planner.py:81-102``) becomes exactly one pull of K and one of V in its coalesced
stage; the Delta-matching guarantees each GPU reads from at most ``degree`` peers
and is read by at most ``degree`` peers per stage.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

from . import native
from .distributor import chunk_placement
from .worklist import rank_layout


def _append_merged(pulls, pull):
    """Append (peer, src, dst, n), coalescing with the previous pull when both ranges
    continue contiguously on the same peer (fewer, larger copy-engine transfers)."""
    if pulls:
        pp, ps, pd, pn = pulls[-1]
        peer, src, dst, n = pull
        if pp == peer and ps + pn == src and pd + pn == dst:
            pulls[-1] = (pp, ps, pd, pn + n)
            return
    pulls.append(pull)


class SymmetricExchange:
    def __init__(self, result, rank: int, cfg, device, group=None, layouts=None):
        self.rank = rank
        self.world = result.assignment.n_workers
        self.device = device
        self.group = group or dist.group.WORLD
        H, D = cfg.kv_heads, cfg.head_dim
        layouts = layouts or [rank_layout(result, r) for r in range(self.world)]
        self.layouts = layouts
        me = layouts[rank]
        t_max = max(l.tokens for l in layouts)
        r_max = max(max(l.recv_tokens for l in layouts), 1)
        self.kv = symm.empty(2 * t_max * H * D, dtype=torch.bfloat16, device=device).view(2, t_max, H, D)
        self.part = symm.empty(2 * r_max * H * D, dtype=torch.float32, device=device).view(2, r_max, H, D)
        self.h_kv = symm.rendezvous(self.kv, self.group)
        self.h_part = symm.rendezvous(self.part, self.group)
        self.peer_kv = [self.h_kv.get_buffer(p, (2, t_max, H, D), torch.bfloat16)
                        for p in range(self.world)]
        self.peer_part = [self.h_part.get_buffer(p, (2, r_max, H, D), torch.float32)
                          for p in range(self.world)]
        # Readiness flags: [channel][src rank] int32 words in symmetric memory, written by
        # the peers' stream front ends (native.stream_signal) and waited on locally.
        self.flags = symm.empty(self.N_CHANNELS * self.world, dtype=torch.int32, device=device)
        self.flags.zero_()
        self.h_flags = symm.rendezvous(self.flags, self.group)
        self.flag_base = [int(a) for a in self.h_flags.buffer_ptrs]
        self.epoch = [0] * self.N_CHANNELS
        torch.cuda.synchronize(device)
        dist.barrier(group=self.group)                  # every rank's flags are zero
        # Pulls from different peers go to different streams so several copy engines run
        # at once (one stream serialises every copy on one engine).
        self.copy_streams = [torch.cuda.Stream(device=device) for _ in range(min(4, max(self.world - 1, 1)))]
        self.kv_row_bytes = 2 * H * D * 2          # K and V, bf16
        self.part_row_bytes = H * D * 4            # one fp32 partial row (dK or dV)
        self.t_local = me.tokens
        self.r_local = me.recv_tokens
        # forward pulls, per coalesced stage: (peer, src_row in peer's K/V, dst_row in my arena, n)
        # Every chunk is pulled from its owner's buffer: over NVSwitch any peer is one hop
        # away, so a relay edge (ring / ByteScale plans) only fixes *when* it arrives.
        owner = chunk_placement(result.assignment, result.units)
        self.stage_pulls: list[list[tuple[int, int, int, int]]] = []
        for s, stage in enumerate(result.plan.stages):
            pulls: list[tuple[int, int, int, int]] = []
            for e in stage:
                if e.dst != rank:
                    continue
                for c in e.chunks:
                    if me.recv_stage.get(c) == s:
                        o = owner[c]
                        _append_merged(pulls, (o, layouts[o].offset[c],
                                               me.recv_offset[c], me.chunk_tokens[c]))
            self.stage_pulls.append(pulls)

    # ------------------------------------------------------------------ forward (K5)
    def publish_kv(self, k, v):
        """Copy this rank's K/V into its symmetric buffer (compute stream)."""
        self.kv[0, :self.t_local].copy_(k, non_blocking=True)
        self.kv[1, :self.t_local].copy_(v, non_blocking=True)

    N_CHANNELS = 4          # kv ready, kv consumed, partials ready, partials consumed
    BARRIER = os.environ.get("FCPB_BARRIER", "flags")   # "kernel": torch's barrier (A/B only)

    def barrier(self, which: str = "kv", channel: int = 0):
        """All-rank barrier on the current stream.  Stream memory operations, not a kernel:
        every rank writes epoch e into each peer's flag word [channel][me], then waits for
        its own [channel][p] words to reach e.  A barrier kernel cannot become resident
        while a persistent attention kernel fills every SM's shared memory (K2 uses all
        227 KB), so it used to wait for the whole launch (C2 at N=4: the partial returns
        started 2 ms late)."""
        if self.BARRIER == "kernel":
            (self.h_kv if which == "kv" else self.h_part).barrier(channel=channel)
            return
        self.signal_all(which, channel)
        cur = torch.cuda.current_stream(self.device)
        for p in range(self.world):
            if p != self.rank:
                self.wait_peer(which, channel, p, cur)

    def _channel(self, which: str, channel: int) -> int:
        return (0 if which == "kv" else 2) + channel

    def signal_all(self, which: str, channel: int) -> None:
        """Open a new epoch on the channel and tell every peer (current stream)."""
        ch = self._channel(which, channel)
        self.epoch[ch] += 1
        cur = torch.cuda.current_stream(self.device)
        w, me = self.world, self.rank
        for p in range(w):
            if p != me:
                native.stream_signal(self.flag_base[p] + 4 * (ch * w + me), self.epoch[ch], cur)

    def wait_peer(self, which: str, channel: int, peer: int, stream) -> None:
        """Work queued on `stream` after this waits for peer's signal of the current epoch."""
        ch = self._channel(which, channel)
        native.stream_wait(self.flag_base[self.rank] + 4 * (ch * self.world + peer), self.epoch[ch], stream)

    FANOUT_BYTES = 64 << 20

    def _fanout(self, copies, nbytes, pre=None):
        """Run (peer, fn) copies with one stream per peer (mod the copy-stream count), ordered
        after the current stream's prior work; the current stream then waits for all.
        Measured on C2/C4 at N=4: fan-out lifts large exchanges (C4 returns 411 -> 483 GB/s)
        but the fork/join costs more than it gains below ~64 MB (C2 pulls 260 -> 171 GB/s),
        so small copy sets stay on the current stream.
        `pre(peer, stream)`, when given, runs once per peer on the stream that carries its
        copies, before the first of them (a per-peer readiness wait)."""
        cur = torch.cuda.current_stream(self.device)
        seen = set()
        if nbytes < self.FANOUT_BYTES or len(self.copy_streams) == 1:
            for peer, fn in copies:
                if pre is not None and peer not in seen:
                    pre(peer, cur)
                    seen.add(peer)
                fn()
            return
        used = set()
        for peer, fn in copies:
            i = peer % len(self.copy_streams)
            cs = self.copy_streams[i]
            if i not in used:
                cs.wait_stream(cur)
                used.add(i)
            if pre is not None and peer not in seen:
                pre(peer, cs)
                seen.add(peer)
            with torch.cuda.stream(cs):
                fn()
        for i in used:
            cur.wait_stream(self.copy_streams[i])

    def pull_stage(self, s: int, k_recv, v_recv):
        """Copy-engine pulls of stage s's KV chunks into the receive arena (ordered on the
        current stream)."""
        def pull(peer, src, dst, n):
            pk = self.peer_kv[peer]
            k_recv[dst:dst + n].copy_(pk[0, src:src + n], non_blocking=True)
            v_recv[dst:dst + n].copy_(pk[1, src:src + n], non_blocking=True)
        pulls = self.stage_pulls[s]
        self._fanout([(peer, (lambda a=(peer, src, dst, n): pull(*a))) for peer, src, dst, n in pulls],
                     sum(n for _, _, _, n in pulls) * self.kv_row_bytes)

    # ------------------------------------------------------------------ backward (K6)
    def partial_views(self):
        """dK/dV partial buffers for the received chunks (the dK/dV kernel writes them)."""
        if self.r_local == 0:
            return None, None
        return self.part[0, :self.r_local], self.part[1, :self.r_local]

    def pull_returns(self, returns, staging_k, staging_v, staging_rows, per_peer_ready=False):
        """Owner side: pull every consumer's partial of my chunks (``exchange.owner_returns``)
        into staging rows.  per_peer_ready: each consumer's pulls wait only for that
        consumer's "partials ready" signal (``signal_all("part", 0)``), not for all ranks."""
        def pull(peer, src, r, n):
            pp = self.peer_part[peer]
            staging_k[r:r + n].copy_(pp[0, src:src + n], non_blocking=True)
            staging_v[r:r + n].copy_(pp[1, src:src + n], non_blocking=True)
        copies = []
        for t in returns:               # chunk t.chunk of mine, consumed by t.peer
            a = (t.peer, self.layouts[t.peer].recv_offset[t.chunk], staging_rows[(t.chunk, t.peer)],
                 t.tokens)
            copies.append((t.peer, (lambda a=a: pull(*a))))
        pre = (lambda peer, st: self.wait_peer("part", 0, peer, st)) if per_peer_ready else None
        self._fanout(copies, sum(t.tokens for t in returns) * 2 * self.part_row_bytes, pre)
