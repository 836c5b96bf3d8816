"""K5/K6 transport: copy-engine pulls from peer-mapped memory over NVLink.

Measured on the B200 box: NCCL grouped send/recv moved the FCP stages at ~45 GB/s
(2 MB messages, and its kernels compete with the persistent attention kernels for
SMs), while ``cudaMemcpyAsync`` pulls from a peer's mapped buffer reach ~250 GB/s
per direction for the same 2 MB chunks with *no* SM use.  Per the north star
("NCCL grouped send/recv, or in-kernel P2P, whichever measures faster") the executor
uses the pulls.

The plan -> copy lists translation is pure host code (``stage_pulls``, ``return_pulls``),
tested on CPU against the reference's arrival semantics (``simulator.py:112-133``).

Buffers (one peer-memory region each, the same size on every rank; ``ipc.IpcRegion`` --
``fcpb_ipc_*`` in the C ABI -- or torch symmetric memory with FCPB_TRANSPORT=symm):

* ``kv``   bf16 [2, T_max, Hkv, D] -- each rank's own K and V planes.  The executor hands
  these planes out as its K/V input buffers, so writing K/V there costs no publish copy.
* ``part`` fp32 [2, R_max, Hkv, D] -- dK/dV partials of the chunks a rank *received*
  (written directly by the dK/dV kernel), pulled back by the chunk owners.
* ``flags`` int32 [4, world] -- readiness words written by the peers' streams
  (``FlagBarrier``).

Every pull of a run of rows moves its K rows and V rows (or dK and dV partial rows) as ONE
2-D copy (``fcpb_copy_2d``): the two planes of the source region and of the destination
arena sit at fixed pitches.

Ordering: an all-rank barrier after the K/V are in place (everyone's K/V is readable), after
the forward pulls (K/V may be overwritten next step), after the partials are written,
and after the return pulls.  The barrier is stream memory operations on the flag words
(``fcpb_stream_signal`` / ``fcpb_stream_wait``), executed without an SM.  Each plan edge
(reference ``planner.py:81-102``) becomes exactly one pull in its coalesced stage; the
Delta-matching guarantees each GPU reads from at most ``degree`` peers and is read by at
most ``degree`` peers per stage.
"""

from __future__ import annotations

import os
from typing import NamedTuple

import torch
import torch.distributed as dist

from . import native
from .distributor import chunk_placement
from .worklist import rank_layout


class Pull(NamedTuple):
    peer: int      # rank whose region is read
    src: int       # first row in the peer's region plane
    dst: int       # first row in my destination plane
    rows: int


def _append_merged(pulls: list, pull: Pull) -> None:
    """Append a pull, coalescing it with the previous one when both ranges continue
    contiguously on the same peer (fewer, larger copy-engine transfers)."""
    if pulls:
        last = pulls[-1]
        if last.peer == pull.peer and last.src + last.rows == pull.src and last.dst + last.rows == pull.dst:
            pulls[-1] = Pull(last.peer, last.src, last.dst, last.rows + pull.rows)
            return
    pulls.append(pull)


def stage_pulls(result, rank: int, layouts=None, owner=None) -> list[list[Pull]]:
    """K5, per coalesced stage: the pulls that fill this rank's receive arena.  Every chunk
    that arrives in stage s (``RankLayout.recv_stage``, the reference's arrival stage,
    ``simulator.py:112-133``) is read from its *owner's* K/V plane, even when the plan's
    edge comes from a relay (ring / ByteScale): over NVSwitch every peer is one hop away,
    so a relay edge only fixes when the chunk arrives.  Pure host code."""
    world = result.assignment.n_workers
    layouts = layouts or [rank_layout(result, r) for r in range(world)]
    owner = owner or chunk_placement(result.assignment, result.units)
    me = layouts[rank]
    out: list[list[Pull]] = []
    for s, stage in enumerate(result.plan.stages):
        pulls: list[Pull] = []
        for e in stage:
            if e.dst != rank:
                continue
            for c in e.chunks:
                if me.recv_stage.get(c) == s:
                    o = owner[c]
                    _append_merged(pulls, Pull(o, layouts[o].offset[c], me.recv_offset[c], me.chunk_tokens[c]))
        out.append(pulls)
    return out


def return_pulls(returns, layouts, staging_rows) -> list[Pull]:
    """K6, owner side: one pull per (my chunk, consuming rank) -- ``exchange.owner_returns``
    -- from the consumer's partial plane (the chunk's receive-arena row there) into my
    staging rows ``staging_rows[(chunk, consumer)]``.  Pure host code."""
    out: list[Pull] = []
    for t in returns:
        _append_merged(out, Pull(t.peer, layouts[t.peer].recv_offset[t.chunk],
                                 staging_rows[(t.chunk, t.peer)], t.tokens))
    return out


# ---------------------------------------------------------------------------- regions
class _Regions:
    """One peer-memory buffer per rank: ``local`` (a torch view of mine) and ``peers[p]``
    (a view of rank p's), through the C-ABI IPC regions or torch symmetric memory."""

    def __init__(self, numel: int, dtype, shape, device, group, backend: str):
        self.backend = backend
        self._keep = None
        if backend == "symm":
            import torch.distributed._symmetric_memory as symm
            buf = symm.empty(numel, dtype=dtype, device=device)
            h = symm.rendezvous(buf, group)
            world = dist.get_world_size(group)
            self.local = buf.view(shape)
            self.peers = [h.get_buffer(p, tuple(shape), dtype) for p in range(world)]
            self.ptrs = [int(x) for x in h.buffer_ptrs]
            self._keep = (buf, h)
        else:
            from .ipc import IpcRegion
            esz = torch.empty((), dtype=dtype).element_size()
            reg = IpcRegion(numel * esz, device)
            regions = reg.exchange(group)
            self.local = reg.tensor(dtype, shape)
            self.peers = [r.tensor(dtype, shape) for r in regions]
            self.ptrs = [r.ptr for r in regions]
            self._keep = regions

    def close_peers(self) -> None:
        """Unmap the peers' regions (first half of a collective close)."""
        if self.backend == "symm" or self._keep is None:
            return
        for r in self._keep:
            if r._opened:
                r.close()
        self.peers = []

    def free_local(self) -> None:
        """Free this rank's region (after every peer has unmapped it)."""
        if self.backend == "symm" or self._keep is None:
            self._keep = None
            return
        for r in self._keep:
            if r._owned:
                r.close()
        self._keep = None
        self.local = None


def close_regions(regions, group) -> None:
    """Collective release of peer-memory regions: every rank unmaps its peers' regions, a
    barrier, then every rank frees its own (a region must not be freed while a peer still
    has it mapped)."""
    torch.cuda.synchronize()
    for r in regions:
        r.close_peers()
    dist.barrier(group=group)
    for r in regions:
        r.free_local()


TRANSPORT = os.environ.get("FCPB_TRANSPORT", "ipc")   # "symm": torch symmetric memory (A/B)


class FlagBarrier:
    """All-rank barriers and per-peer readiness signals on int32 flag words in peer memory,
    executed by the streams' front ends (``fcpb_stream_signal`` / ``fcpb_stream_wait``, i.e.
    cuStreamWriteValue32 / cuStreamWaitValue32 with monotonically increasing epochs) -- no
    kernel, so no SM: a barrier kernel cannot become resident while a persistent attention
    kernel fills every SM's shared memory (K2 uses all 227 KB) and used to wait for whole
    launches (C3 at N=4: 657 -> 629 ms when these flags replaced it).
    Flag word [channel][src] of rank r is written by rank src."""

    def __init__(self, channels: int, device, group, backend: str = TRANSPORT):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        self.channels = channels
        reg = _Regions(channels * self.world, torch.int32, (channels * self.world,), device, group, backend)
        reg.local.zero_()
        self.base = reg.ptrs
        self._reg = reg
        self.epoch = [0] * channels

    def signal_all(self, ch: int, stream=None) -> None:
        """Open a new epoch on channel ch and tell every peer (after `stream`'s prior work)."""
        stream = stream or torch.cuda.current_stream(self.device)
        self.epoch[ch] += 1
        w, me = self.world, self.rank
        for p in range(w):
            if p != me:
                native.stream_signal(self.base[p] + 4 * (ch * w + me), self.epoch[ch], stream)

    def wait_peer(self, ch: int, peer: int, stream) -> None:
        """Work queued on `stream` after this waits for peer's signal of the current epoch."""
        native.stream_wait(self.base[self.rank] + 4 * (ch * self.world + peer), self.epoch[ch], stream)

    def barrier(self, ch: int, stream=None) -> None:
        stream = stream or torch.cuda.current_stream(self.device)
        self.signal_all(ch, stream)
        for p in range(self.world):
            if p != self.rank:
                self.wait_peer(ch, p, stream)


class SymmetricExchange:
    TRANSPORT = TRANSPORT

    def __init__(self, result, rank: int, cfg, device, group=None, layouts=None):
        self.rank = rank
        self.world = result.assignment.n_workers
        self.device = device
        self.group = group or dist.group.WORLD
        H, D = cfg.kv_heads, cfg.head_dim
        layouts = layouts or [rank_layout(result, r) for r in range(self.world)]
        self.layouts = layouts
        me = layouts[rank]
        self.t_max = t_max = max(max(l.tokens for l in layouts), 1)
        self.r_max = r_max = max(max(l.recv_tokens for l in layouts), 1)
        be = self.TRANSPORT
        kv = _Regions(2 * t_max * H * D, torch.bfloat16, (2, t_max, H, D), device, self.group, be)
        part = _Regions(2 * r_max * H * D, torch.float32, (2, r_max, H, D), device, self.group, be)
        self.kv, self.peer_kv = kv.local, kv.peers
        self.part, self.peer_part = part.local, part.peers
        # Readiness flags: [channel][src rank] int32 words in peer memory
        self.flags = FlagBarrier(self.N_CHANNELS, device, self.group, be)
        self._regions = (kv, part)
        torch.cuda.synchronize(device)
        dist.barrier(group=self.group)                  # every rank's flags are zero
        # Pulls from different peers go to different streams so several copy engines run
        # at once (one stream serialises every copy on one engine).
        self.copy_streams = [torch.cuda.Stream(device=device) for _ in range(min(4, max(self.world - 1, 1)))]
        self.kv_row_bytes = 2 * H * D * 2          # K and V, bf16
        self.part_row_bytes = H * D * 4            # one fp32 partial row (dK or dV)
        self.t_local = me.tokens
        self.r_local = me.recv_tokens
        self.stage_pulls = stage_pulls(result, rank, layouts)
        self.publish_copies = 0                   # K/V publish copies issued (0 when zero-copy)

    def close(self) -> None:
        """Release the exchange's peer-memory regions (collective: every rank calls it)."""
        if self._regions is None:
            return
        close_regions(list(self._regions) + [self.flags._reg], self.group)
        self._regions = None

    # ------------------------------------------------------------------ forward (K5)
    def kv_views(self):
        """This rank's K and V planes in the exchange region ([T, Hkv, D] each, contiguous):
        the executor's K/V input buffers."""
        return self.kv[0, :self.t_local], self.kv[1, :self.t_local]

    def publish_kv(self, k, v):
        """Make this rank's K/V readable by the peers (compute stream): free when the caller
        wrote them into ``kv_views()``, otherwise one copy each."""
        kk, vv = self.kv_views()
        if k.data_ptr() != kk.data_ptr():
            kk.copy_(k, non_blocking=True)
            self.publish_copies += 1
        if v.data_ptr() != vv.data_ptr():
            vv.copy_(v, non_blocking=True)
            self.publish_copies += 1

    N_CHANNELS = 4          # kv ready, kv consumed, partials ready, partials consumed
    BARRIER = os.environ.get("FCPB_BARRIER", "flags")   # "kernel": torch's barrier (symm only, A/B)

    def barrier(self, which: str = "kv", channel: int = 0):
        """All-rank barrier on the current stream (``FlagBarrier``)."""
        if self.BARRIER == "kernel" and self.TRANSPORT == "symm":
            self._regions[0 if which == "kv" else 1]._keep[1].barrier(channel=channel)
            return
        self.flags.barrier(self._channel(which, channel))

    def _channel(self, which: str, channel: int) -> int:
        return (0 if which == "kv" else 2) + channel

    def signal_all(self, which: str, channel: int) -> None:
        """Open a new epoch on the channel and tell every peer (current stream)."""
        self.flags.signal_all(self._channel(which, channel))

    def wait_peer(self, which: str, channel: int, peer: int, stream) -> None:
        """Work queued on `stream` after this waits for peer's signal of the current epoch."""
        self.flags.wait_peer(self._channel(which, channel), peer, stream)

    FANOUT_BYTES = 64 << 20

    def _fanout(self, pulls, nbytes, fn, pre=None):
        """Issue fn(pull) for every pull, with one stream per peer (mod the copy-stream
        count), ordered after the current stream's prior work; the current stream then
        waits for all.  Measured on C2/C4 at N=4: fan-out lifts large exchanges (C4 returns
        411 -> 483 GB/s) but the fork/join costs more than it gains below ~64 MB (C2 pulls
        260 -> 171 GB/s), so small copy sets stay on the current stream.
        `pre(peer, stream)`, when given, runs once per peer on the stream that carries its
        copies, before the first of them (a per-peer readiness wait)."""
        cur = torch.cuda.current_stream(self.device)
        seen = set()
        if nbytes < self.FANOUT_BYTES or len(self.copy_streams) == 1:
            for p in pulls:
                if pre is not None and p.peer not in seen:
                    pre(p.peer, cur)
                    seen.add(p.peer)
                fn(p, cur)
            return
        used = set()
        for p in pulls:
            i = p.peer % len(self.copy_streams)
            cs = self.copy_streams[i]
            if i not in used:
                cs.wait_stream(cur)
                used.add(i)
            if pre is not None and p.peer not in seen:
                pre(p.peer, cs)
                seen.add(p.peer)
            fn(p, cs)
        for i in used:
            cur.wait_stream(self.copy_streams[i])

    @staticmethod
    def _planes(dst):
        """(base pointer, plane pitch in bytes, row bytes) of a [2, R, H, D] destination."""
        assert dst.dim() == 4 and dst.shape[0] == 2 and dst.is_contiguous()
        row = dst.shape[2] * dst.shape[3] * dst.element_size()
        return dst.data_ptr(), dst.shape[1] * row, row

    def pull_stage(self, s: int, kv_recv):
        """Copy-engine pulls of stage s's KV chunks into the receive arena ``kv_recv``
        ([2, R, Hkv, D] bf16: the K plane then the V plane), one 2-D copy per merged run
        (ordered on the current stream)."""
        pulls = self.stage_pulls[s]
        if not pulls:                  # e.g. a rank that receives nothing in this stage
            return
        base, dpitch, row = self._planes(kv_recv)
        spitch = self.t_max * row

        def pull(p, stream):
            native.copy_2d(base + p.dst * row, dpitch, self.peer_kv[p.peer].data_ptr() + p.src * row,
                           spitch, p.rows * row, 2, stream)
        self._fanout(pulls, sum(p.rows for p in pulls) * self.kv_row_bytes, pull)

    GATHER_CTAS = 2 * 148       # two 512-thread CTAs per SM: 128 KB of peer loads in flight per SM

    def gather_segments(self, kv_recv) -> list[tuple[int, int, int]]:
        """Every stage's pulls as (dst, src, bytes) ranges for the pull kernel: one range per
        plane of each merged run, split at ``native.gather_seg_bytes()``."""
        base, dpitch, row = self._planes(kv_recv)
        spitch = self.t_max * row
        step = native.gather_seg_bytes()
        segs = []
        for pulls in self.stage_pulls:
            for p in pulls:
                n = p.rows * row
                for plane in range(2):
                    d = base + plane * dpitch + p.dst * row
                    s_ = self.peer_kv[p.peer].data_ptr() + plane * spitch + p.src * row
                    for o in range(0, n, step):
                        segs.append((d + o, s_ + o, min(step, n - o)))
        return segs

    def gather_all(self, kv_recv, stream=None) -> None:
        """All stages' K/V pulls as one pull-kernel launch on `stream` (SM loads from the
        peers' regions over NVLink, ``fcpb_gather_copy``).  The segment table is built once
        per receive arena and kept on the device."""
        key = kv_recv.data_ptr()
        if getattr(self, "_gather_key", None) != key:
            segs = self.gather_segments(kv_recv)
            self._gather_tab = torch.tensor(segs, dtype=torch.int64).reshape(-1, 3).to(self.device)
            self._gather_key = key
        if self._gather_tab.shape[0]:
            native.gather_copy(self._gather_tab, self.GATHER_CTAS,
                               stream or torch.cuda.current_stream(self.device))

    # ------------------------------------------------------------------ backward (K6)
    def partial_views(self):
        """dK/dV partial buffers for the received chunks (the dK/dV kernel writes them)."""
        if self.r_local == 0:
            return None, None
        return self.part[0, :self.r_local], self.part[1, :self.r_local]

    def pull_returns(self, returns, staging, staging_rows, per_peer_ready=False):
        """Owner side: pull every consumer's partial of my chunks (``exchange.owner_returns``)
        into ``staging`` ([2, rows, Hkv, D] fp32: dK then dV plane), one 2-D copy per merged
        run.  per_peer_ready: each consumer's pulls wait only for that consumer's "partials
        ready" signal (``signal_all("part", 0)``), not for all ranks."""
        pulls = return_pulls(returns, self.layouts, staging_rows)
        if not pulls:
            return
        base, dpitch, row = self._planes(staging)
        spitch = self.r_max * row

        def pull(p, stream):
            native.copy_2d(base + p.dst * row, dpitch, self.peer_part[p.peer].data_ptr() + p.src * row,
                           spitch, p.rows * row, 2, stream)
        pre = (lambda peer, st: self.wait_peer("part", 0, peer, st)) if per_peer_ready else None
        self._fanout(pulls, sum(p.rows for p in pulls) * 2 * self.part_row_bytes, pull, pre)
