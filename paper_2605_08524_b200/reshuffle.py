"""the transparent reshuffler -- user layout <-> FCP layout over NVLink.

A model keeps its activations in a *user layout*: each rank holds a contiguous share of
the batch's chunks.  This is the reference's ``default_contiguous_layout``
(``simulator.py:279-291``): chunks fill ranks in unit order; any other chunk -> rank map
can be passed instead.  FCP computes in the plan's layout (``worklist.rank_layout``).  The
reshuffler moves every row of Q/K/V/dO into the FCP layout before the attention step and
every row of O/LSE/dQ/dK/dV back afterwards, so the op drops into a model without
touching its data loader.

* Plan (host, every rank, deterministic): for each chunk a rank owns in the destination
  layout, pull it from the rank that holds it in the source layout.  Contiguous runs on
  the same peer are merged.  A chunk whose two owners coincide is a local copy.  The
  bytes moved are exactly the reference's ``reshuffle_cost`` accounting
  (``simulator.py:294-342``); ``tests/test_reshuffle.py`` checks that.
* Transport (GPU): one peer-memory byte buffer (``p2p._Regions``: a C-ABI IPC region)
  with one contiguous region per tensor of a call, so each call is:
  1. one contiguous publish per tensor;
  2. one flag barrier (stream memory operations, no kernel);
  3. copy-engine pulls of whole contiguous row runs from the peers' regions, straight into
     the output tensors;
  4. one flag barrier.
  This is the same transport as the KV exchange (``p2p.py``).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import native
from .costmodel import ModelConfig
from .distributor import chunk_placement
from .errors import ConsistencyError, ParameterError
from .pipeline import ScheduleResult
from .simmodel import default_contiguous_layout
from .worklist import rank_layout


@dataclass
class UserLayout:
    """One rank's share of the user layout: its chunks in user order and their rows."""
    rank: int
    chunks: list
    offset: dict
    tokens: int


def user_layouts(result: ScheduleResult, initial_layout=None) -> list[UserLayout]:
    """Per-rank user layouts.  ``initial_layout``: ChunkKey -> rank (default: the
    reference's contiguous layout); rows follow unit order, then member order."""
    n = result.assignment.n_workers
    init = initial_layout if initial_layout is not None else default_contiguous_layout(result.units, n)
    keys = {c.key for u in result.units for c in u.members}
    if set(init) != keys:
        raise ConsistencyError("initial layout covers a different chunk set")
    out = [UserLayout(r, [], {}, 0) for r in range(n)]
    for u in result.units:
        for c in u.members:
            r = init[c.key]
            if not 0 <= r < n:
                raise ParameterError(f"initial layout puts {c.key} on rank {r} (N={n})")
            lay = out[r]
            lay.offset[c.key] = lay.tokens
            lay.chunks.append(c.key)
            lay.tokens += c.token_count
    return out


def _append(pulls, pull):
    """Append (peer, src_row, dst_row, n), merging with a contiguous predecessor."""
    if pulls:
        pp, ps, pd, pn = pulls[-1]
        peer, src, dst, n = pull
        if pp == peer and ps + pn == src and pd + pn == dst:
            pulls[-1] = (pp, ps, pd, pn + n)
            return
    pulls.append(pull)


@dataclass
class ReshufflePlan:
    """Row moves of one rank, both directions: (peer, src_row, dst_row, rows)."""
    rank: int
    to_fcp: list
    from_fcp: list
    user_tokens: int
    fcp_tokens: int


def reshuffle_plans(result: ScheduleResult, initial_layout=None) -> list[ReshufflePlan]:
    n = result.assignment.n_workers
    users = user_layouts(result, initial_layout)
    fcps = [rank_layout(result, r) for r in range(n)]
    user_of = {c: u.rank for u in users for c in u.chunks}
    owner = chunk_placement(result.assignment, result.units)
    tokens = result.deps.chunk_tokens
    plans = []
    for r in range(n):
        to_f: list = []
        for c in fcps[r].chunks:              # rows this rank needs in the FCP layout
            src = user_of[c]
            _append(to_f, (src, users[src].offset[c], fcps[r].offset[c], tokens[c]))
        back: list = []
        for c in users[r].chunks:             # rows this rank needs back in its user layout
            src = owner[c]
            _append(back, (src, fcps[src].offset[c], users[r].offset[c], tokens[c]))
        plans.append(ReshufflePlan(r, to_f, back, users[r].tokens, fcps[r].tokens))
    return plans


def moved_bytes(plans: list[ReshufflePlan], bytes_per_token: int) -> tuple[list[int], list[int]]:
    """(out_bytes, in_bytes) per rank of the to-FCP direction, excluding local copies --
    the quantity ``simulator.reshuffle_cost`` reports."""
    n = len(plans)
    out, inn = [0] * n, [0] * n
    for p in plans:
        for peer, _, _, rows in p.to_fcp:
            if peer != p.rank:
                inn[p.rank] += rows * bytes_per_token
                out[peer] += rows * bytes_per_token
    return out, inn


def apply_pulls(pulls, sources, dst):
    """Reference semantics of one direction (CPU tests): dst[d:d+n] = sources[peer][s:s+n]."""
    for peer, s, d, n in pulls:
        dst[d:d + n] = sources[peer][s:s + n]
    return dst


class Reshuffler:
    """Collective user <-> FCP layout moves for one rank (call on every rank, same order).

    ``max_row_bytes`` bounds the per-token bytes of one call.  The default covers Q, K, V,
    dO in and O, LSE, dQ, dK, dV out for ``cfg``.
    """

    def __init__(self, result: ScheduleResult, rank: int, cfg: ModelConfig, device,
                 initial_layout=None, group=None, max_row_bytes: int | None = None):
        import torch.distributed as dist
        from .p2p import FlagBarrier, _Regions, TRANSPORT
        self.rank = rank
        self.world = result.assignment.n_workers
        self.device = torch.device(device)
        self.plans = reshuffle_plans(result, initial_layout)
        self.plan = self.plans[rank]
        from .distributor import chunk_placement
        owner = chunk_placement(result.assignment, result.units)
        self._resident = {c for c in user_layouts(result, initial_layout)[rank].chunks if owner[c] == rank}
        H, Hk, D = cfg.q_heads, cfg.kv_heads, cfg.head_dim
        self.row_cap = max_row_bytes or ((2 * H + 2 * Hk) * D * 2 + 4 * H)
        self.t_max = max(max(max(p.user_tokens, p.fcp_tokens) for p in self.plans), 1)
        group = group or dist.group.WORLD
        self._group = group
        reg = _Regions(self.t_max * self.row_cap, torch.uint8, (self.t_max * self.row_cap,),
                       self.device, group, TRANSPORT)
        self.buf, self.peer, self._reg = reg.local, reg.peers, reg
        self.flags = FlagBarrier(2, self.device, group)
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)                       # every rank's flags are zero
        self.bytes_moved = 0
        self._tabs = {}            # gather segment tables per move shape (_gather)

    def _move(self, tensors, pulls, rows_in: int, rows_out: int, outs=None, remote_stream=None,
              defer_remote: bool = False):
        """Move rows of every tensor along `pulls`.  Rows that stay on this rank are copied
        straight from the inputs on the current stream; the others go through the peers'
        regions (publish, flag barrier, copy-engine pulls, flag barrier).  With
        `remote_stream` that remote part runs there, concurrently with whatever the caller
        queues next on the current stream, and the method returns (outs, event): the
        outputs are complete once the current stream has also waited for the event.
        defer_remote (with remote_stream): return (outs, start) after the local copies;
        start() enqueues the remote part and returns the event, so the caller can enqueue its
        own work on the current stream first (the remote part's ~40 host-side copy launches
        would otherwise hold back the host's next launch: 0.4 ms, scripts/forward_user_probe.py)."""
        widths, elems = [], []
        for t in tensors:
            if t.shape[0] != rows_in:
                raise ParameterError(f"tensor has {t.shape[0]} rows, layout has {rows_in}")
            row = 1
            for x in t.shape[1:]:
                row *= x
            elems.append(row)
            widths.append(row * t.element_size())
        if sum(widths) > self.row_cap:
            raise ParameterError(f"{sum(widths)} bytes per row exceed the reshuffler's {self.row_cap}")
        if outs is None:
            outs = [torch.empty((rows_out,) + tuple(t.shape[1:]), dtype=t.dtype, device=self.device)
                    for t in tensors]
        flat_in = [t.contiguous().reshape(rows_in, e) for t, e in zip(tensors, elems)]
        flat_out = [o.view(rows_out, e) for o, e in zip(outs, elems)]
        self._mark("begin")
        # rows that stay here: direct copies, all of them in one gather-kernel launch (one
        # torch copy per (tensor, run) left the GPU waiting on the host's launches: 0.64 ms
        # for C2's 45 local runs at N=2, scripts/reshuffle_probe.py)
        m = len(tensors)      # bases: outputs 0..m-1, inputs m..2m-1, peer regions 2m..
        bases = ([o.data_ptr() for o in flat_out] + [t.data_ptr() for t in flat_in] +
                 [x.data_ptr() for x in self.peer])
        local = [(i, d * w, m + i, s0 * w, n * w) for i, w in enumerate(widths)
                 for peer, s0, d, n in pulls if peer == self.rank]
        if not self._gather(local, bases, torch.cuda.current_stream(self.device)):
            for src, dst in zip(flat_in, flat_out):
                for peer, s0, d, n in pulls:
                    if peer == self.rank:
                        dst[d:d + n].copy_(src[s0:s0 + n], non_blocking=True)
        # one contiguous region per tensor (capacity t_max rows each): publish and pulls are
        # plain contiguous copies and the pulls land directly in the outputs (no unpack)
        region, acc = [], 0
        for w in widths:
            region.append(acc)
            acc += self.t_max * w
        cur = torch.cuda.current_stream(self.device)
        st = remote_stream or cur
        self._mark("local_copies", cur)
        # the remote part waits for the inputs and the local copies, not for whatever the
        # caller enqueues on the current stream before calling a deferred start()
        local_done = torch.cuda.Event()
        local_done.record(cur)

        def remote_part():
            if remote_stream is not None:
                remote_stream.wait_event(local_done)
            with torch.cuda.stream(st):
                for src, w, off in zip(flat_in, widths, region):                # publish
                    dst = self.buf[off:off + rows_in * w]
                    if src.data_ptr() == dst.data_ptr():    # written in place (input_views)
                        continue
                    dst.view(rows_in, w).copy_(src.view(torch.uint8), non_blocking=True)
                self._mark("published", st)
                self.flags.barrier(0, st)              # every rank's rows published
                self._mark("barrier0", st)
                remote = [(i, d * w, 2 * m + peer, off + s0 * w, n * w)
                          for i, (w, off) in enumerate(zip(widths, region)) for peer, s0, d, n in pulls
                          if peer != self.rank]
                self.bytes_moved += sum(x[4] for x in remote)
                # Standalone, the pulls are SM loads over NVLink (the K5 pull kernel, one
                # launch); beside compute (remote_stream) they stay on the copy engines, which
                # need no SM.
                if remote_stream is not None or not self._gather(remote, bases, st):
                    for dst, w, off in zip(flat_out, widths, region):
                        ob = dst.view(torch.uint8)
                        for peer, s0, d, n in pulls:
                            if peer == self.rank:
                                continue
                            ob[d:d + n].copy_(self.peer[peer][off + s0 * w:off + (s0 + n) * w].view(n, w),
                                              non_blocking=True)
                self._mark("pulls", st)
                self.flags.barrier(1, st)              # every pull done: buffers reusable
                self._mark("barrier1", st)
            if remote_stream is None:
                return None
            ev = torch.cuda.Event()
            ev.record(remote_stream)
            for t in list(tensors) + list(outs):
                t.record_stream(remote_stream)
            return ev

        if remote_stream is None:
            remote_part()
            return outs
        if defer_remote:
            return outs, remote_part
        return outs, remote_part()

    # Optional per-phase CUDA-event timeline of _move (scripts/reshuffle_probe.py).
    marks = None

    def _mark(self, name, stream=None):
        if self.marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream or torch.cuda.current_stream(self.device))
            self.marks.append((name, ev))

    def _gather(self, ranges, bases, stream) -> bool:
        """Copy ranges (dst base, dst offset, src base, src offset, bytes) with one
        ``fcpb_gather_copy_based`` launch on `stream`; False (nothing launched) when an address
        or size is not 16-byte aligned.  The segment table depends only on the move's shape, so
        it is uploaded once per shape and reused whatever the tensors' addresses are (a
        per-call upload from freshly pinned memory stalled the host for up to 100 ms)."""
        if not ranges:
            return True
        if len(bases) > 32 or any(b & 15 for b in bases) or any((do | so | n) & 15 for _, do, _, so, n in ranges):
            return False
        key = tuple(ranges)
        cache = self._tabs
        tab = cache.get(key)
        if tab is None:
            import numpy as np
            step = native.gather_seg_bytes()
            r = np.asarray(ranges, dtype=np.int64)
            cnt = (r[:, 4] + step - 1) // step                 # pieces of <= step bytes per range
            idx = np.repeat(np.arange(len(r)), cnt)
            o = (np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)) * step
            segs = np.stack([(r[idx, 0] << 56) | (r[idx, 1] + o), (r[idx, 2] << 56) | (r[idx, 3] + o),
                             np.minimum(step, r[idx, 4] - o)], axis=1)
            tab = torch.from_numpy(np.ascontiguousarray(segs)).to(self.device)   # once per shape
            if len(cache) >= 64:
                cache.clear()
            cache[key] = tab
        native.gather_copy_based(tab, bases, 2 * torch.cuda.get_device_properties(self.device).multi_processor_count,
                                 stream)
        return True

    def input_views(self, specs, rows: int | None = None):
        """Tensors of shapes [rows, *shape] / dtypes ``specs`` that live in this rank's
        region exactly where ``_move`` publishes the same tensor list: a caller that writes its
        user-layout inputs there (e.g. the QKV projection's output) skips the publish copy, a
        same-device copy that would otherwise wait for the SMs the overlapped compute holds.
        Valid until the next move."""
        rows = self.plan.user_tokens if rows is None else rows
        out, off = [], 0
        for shape, dtype in specs:
            esz = torch.empty((), dtype=dtype).element_size()
            e = 1
            for x in shape:
                e *= x
            w = e * esz
            if off + rows * w > self.buf.numel():
                raise ParameterError("input views exceed the reshuffler's region")
            out.append(self.buf[off:off + rows * w].view(dtype).view((rows,) + tuple(shape)))
            off += self.t_max * w
        return out

    def close(self) -> None:
        """Release the region and flags (collective: every rank calls it)."""
        if self._reg is None:
            return
        from .p2p import close_regions
        close_regions([self._reg, self.flags._reg], self._group)
        self._reg = None

    def resident_chunks(self) -> frozenset:
        """Chunks that stay on this rank (their to-FCP pull is local): build the executor with
        ``FcpExecutor(..., resident=rs.resident_chunks())`` so their tiles run while the
        remote pulls of ``FcpExecutor.forward_user`` are in flight."""
        return frozenset(self._resident)

    def to_fcp(self, *tensors):
        """User-layout [T_user, ...] tensors -> FCP-layout [T_fcp, ...] tensors."""
        return self._move(tensors, self.plan.to_fcp, self.plan.user_tokens, self.plan.fcp_tokens)

    def from_fcp(self, *tensors):
        """FCP-layout [T_fcp, ...] tensors -> user-layout [T_user, ...] tensors."""
        return self._move(tensors, self.plan.from_fcp, self.plan.fcp_tokens, self.plan.user_tokens)
