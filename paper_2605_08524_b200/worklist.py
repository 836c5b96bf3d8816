"""H1: turn a ``ScheduleResult`` into per-rank device work lists.

Nothing here exists in the reference: it is the bridge from the plan the
reference computes (``pipeline.py:31-60``) to the tiles its simulator only
times (``simulator.py:73-109``).  For rank ``r``:

* **Layout.**  Local chunks are packed token-major in unit-id order (members
  in unit order); this is the layout of the rank's Q, K, V, O, dO, dQ, dK, dV.
  Remote chunks the rank receives get slots in a *receive arena*, ordered by
  the coalesced stage that delivers them, then by plan edge order
  (``simulator.py:112-133`` defines the arrival stage).
* **Forward waves.**  Wave -1 holds every (Q chunk, KV chunk) tile whose KV is
  local -- the dependency-free prologue; wave s holds tiles whose KV arrives
  with coalesced stage s.  A Q chunk whose tiles span several waves writes one
  fp32 partial (O, LSE) per wave, merged by K3 afterwards; a Q chunk served by
  a single wave writes its final bf16 O directly.
* **Backward.**  dK/dV work is keyed by KV chunk (local or received): the KV
  block iterates over every local Q chunk attending to it.  Received chunks form
  their own launch so their dK/dV partials can travel back along the reversed
  plan edges while the local chunks compute.  dQ is query-stationary: one
  segment per local Q chunk over all of its (by then resident) KV chunks.

Work items are sorted longest-first (LPT over the persistent grid).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .costmodel import tile_token_pairs
from .distributor import chunk_placement
from .errors import ConsistencyError, ParameterError
from .pipeline import ScheduleResult
from .sharding import CAUSAL, ChunkKey
from .simmodel import arrival_stages

TILE = 128
KV_DIAG = 1
KV_RECV = 2
LOCAL_WAVE = -1


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


@dataclass
class RankLayout:
    rank: int
    chunks: list[ChunkKey]
    offset: dict[ChunkKey, int]
    tokens: int
    recv_chunks: list[ChunkKey]
    recv_offset: dict[ChunkKey, int]
    recv_tokens: int
    recv_stage: dict[ChunkKey, int]
    chunk_tokens: dict[ChunkKey, int]
    # received KV chunks some local Q chunk attends to.  FCP plans deliver only these;
    # relay plans (ring / ByteScale) also deliver chunks a rank merely forwards, whose
    # dK/dV partials do not exist and must not be returned.
    consumed: frozenset = frozenset()


@dataclass
class FwdWave:
    stage: int                   # LOCAL_WAVE or the coalesced stage that releases it
    segments: np.ndarray         # int32 [S, 6]: q_off q_len kv_begin kv_end out_row pad
    kvrefs: np.ndarray           # int32 [R, 4]: off len flags pad
    items: np.ndarray            # int32 [I, 2]: seg mblock
    pairs: int                   # visible token pairs (reference tile_token_pairs)
    costs: np.ndarray | None = None   # int64 [I]: 128x128 tiles per item (LPT key)


@dataclass
class FwdPlan:
    waves: list[FwdWave]
    partial_rows: int
    merge_groups: np.ndarray     # int32 [G, 6]: q_off q_len part_begin part_end tok_begin pad
    merge_part_rows: np.ndarray  # int32 [P]
    merged_tokens: int


@dataclass
class BwdLaunch:
    recv: bool
    kvsegs: np.ndarray           # int32 [K, 6]: kv_off kv_len flags q_begin q_end pad
    qrefs: np.ndarray            # int32 [Q, 4]: q_off q_len diag pad
    items: np.ndarray            # int32 [I, 2]: kvseg nblock
    pairs: int
    costs: np.ndarray | None = None   # int64 [I]: 128x128 tiles per item (LPT key)
    kv_keys: list | None = None       # chunk key of every kvseg
    q_keys: list | None = None        # chunk key of every qref
    pair_base: np.ndarray | None = None   # int32 [I]: first dS pair id of the item (build_ds_tiles)


@dataclass
class DqPlan:
    """Query-stationary dQ launch: one segment per local Q chunk listing ALL its KV
    chunks (local and received), same record layout as the forward tables."""
    segments: np.ndarray         # int32 [S, 6]
    kvrefs: np.ndarray           # int32 [R, 4]
    items: np.ndarray            # int32 [I, 2]: seg mblock (LPT order)
    pairs: int
    costs: np.ndarray | None = None   # int64 [I]: 128x128 tiles per item (LPT key)
    q_keys: list | None = None        # chunk key of every segment
    kv_keys: list | None = None       # chunk key of every kvref
    pair_ids: np.ndarray | None = None    # int32: dS pair id of every (item, kv tile), item-major
    pair_off: np.ndarray | None = None    # int32 [I]: first entry of each item in pair_ids


@dataclass
class RankWork:
    layout: RankLayout
    fwd: FwdPlan
    bwd: list[BwdLaunch] = field(default_factory=list)
    pairs: int = 0
    dq: DqPlan | None = None
    ds_pairs: int = 0                 # (kv block, q block) pairs with a materialised dS tile


def rank_layout(result: ScheduleResult, rank: int) -> RankLayout:
    n = result.assignment.n_workers
    if not 0 <= rank < n:
        raise ParameterError(f"rank {rank} outside [0, {n})")
    chunks: list[ChunkKey] = []
    sizes = dict(result.deps.chunk_tokens)
    for u in sorted(result.units, key=lambda u: u.unit_id):
        if result.assignment.worker_of(u.unit_id) == rank:
            chunks += [c.key for c in u.members]
    offset, pos = {}, 0
    for c in chunks:
        offset[c] = pos
        pos += sizes[c]
    where = chunk_placement(result.assignment, result.units)
    arrival = arrival_stages(result.plan.stages, where)
    recv = []
    for s, stage in enumerate(result.plan.stages):
        for e in stage:
            if e.dst == rank:
                for c in e.chunks:
                    if arrival[(c, rank)] == s and c not in recv:
                        recv.append(c)
    roff, rpos = {}, 0
    for c in recv:
        roff[c] = rpos
        rpos += sizes[c]
    rstage = {c: arrival[(c, rank)] for c in recv}
    needed = {kv for q in chunks for kv in result.deps.q_to_kv[q]}
    return RankLayout(rank, chunks, offset, pos, recv, roff, rpos, rstage, sizes,
                      frozenset(c for c in recv if c in needed))


def _kv_location(lay: RankLayout, kv: ChunkKey) -> tuple[int, int, int]:
    """(wave, arena offset, flags) of a KV chunk as seen from this rank."""
    if kv in lay.offset:
        return LOCAL_WAVE, lay.offset[kv], 0
    if kv in lay.recv_offset:
        return lay.recv_stage[kv], lay.recv_offset[kv], KV_RECV
    raise ConsistencyError(f"plan never delivers chunk {kv} to rank {lay.rank}")


def _lpt_order(items):
    """Longest-first (cost, a, b, seq) items over the persistent grid.  The kernels
    combine this item order with the heads (``grid_map``: heads-adjacent, head-major, or
    head-major after a heads-adjacent lead; see ``BlockAttention``)."""
    import os
    if os.environ.get("FCPB_ORDER", "lpt") == "seq":     # experiment knob
        seq_cost: dict[int, int] = {}
        for cost, _, _, seq in items:
            seq_cost[seq] = seq_cost.get(seq, 0) + cost
        return sorted(items, key=lambda t: (-seq_cost[t[3]], t[3], -t[0], t[1], t[2]))
    return sorted(items, key=lambda t: (-t[0], t[1], t[2]))


def build_forward(result: ScheduleResult, lay: RankLayout, fuse_remote: bool = False) -> FwdPlan:
    """Forward waves.  fuse_remote: every received KV chunk goes into one wave released by
    this rank's last arrival stage (one launch, one tail, and at most a local and a remote
    partial per Q chunk) instead of one wave per coalesced stage."""
    deps = result.deps
    causal = deps.mask == CAUSAL
    last_stage = max(lay.recv_stage.values(), default=LOCAL_WAVE)
    # per Q chunk: wave -> ordered kv list
    per_q: dict[ChunkKey, dict[int, list[tuple[int, int, int, int]]]] = {}
    for q in lay.chunks:
        waves: dict[int, list] = {}
        for kv in deps.q_to_kv[q]:
            wave, off, flags = _kv_location(lay, kv)
            if fuse_remote and wave != LOCAL_WAVE:
                wave = last_stage
            if causal and kv == q:
                flags |= KV_DIAG
            waves.setdefault(wave, []).append((off, deps.chunk_tokens[kv], flags, 0))
        per_q[q] = waves

    wave_ids = sorted({w for waves in per_q.values() for w in waves})
    part_rows = 0
    partial_of: dict[ChunkKey, list[tuple[int, int]]] = {}   # q -> [(wave, row)]
    seg_rows: dict[tuple[ChunkKey, int], int] = {}
    for q in lay.chunks:
        waves = per_q[q]
        if len(waves) > 1:
            for w in sorted(waves):
                seg_rows[(q, w)] = part_rows
                partial_of.setdefault(q, []).append((w, part_rows))
                part_rows += deps.chunk_tokens[q]
    out = []
    for w in wave_ids:
        segs, refs, items, pairs = [], [], [], 0
        for q in lay.chunks:
            kvs = per_q[q].get(w)
            if not kvs:
                continue
            qn = deps.chunk_tokens[q]
            begin = len(refs)
            refs += kvs
            for off, kn, flags, _ in kvs:
                pairs += tile_token_pairs(qn, kn, bool(flags & KV_DIAG))
            out_row = seg_rows.get((q, w), -1)
            sidx = len(segs)
            segs.append((lay.offset[q], qn, begin, len(refs), out_row, 0))
            for mb in range(_cdiv(qn, TILE)):
                cost = 0
                for off, kn, flags, _ in kvs:
                    nt = _cdiv(kn, TILE)
                    cost += min(nt, mb + 1) if flags & KV_DIAG else nt
                items.append((cost, sidx, mb, q[0]))
        items = _lpt_order(items)
        out.append(FwdWave(
            w, np.asarray(segs, dtype=np.int32).reshape(-1, 6),
            np.asarray(refs, dtype=np.int32).reshape(-1, 4),
            np.asarray([(s, m) for _, s, m, _ in items], dtype=np.int32).reshape(-1, 2), pairs,
            np.asarray([c for c, _, _, _ in items], dtype=np.int64)))
    groups, rows, tok = [], [], 0
    for q in lay.chunks:
        if q in partial_of:
            begin = len(rows)
            rows += [r for _, r in partial_of[q]]
            groups.append((lay.offset[q], deps.chunk_tokens[q], begin, len(rows), tok, 0))
            tok += deps.chunk_tokens[q]
    return FwdPlan(out, part_rows, np.asarray(groups, dtype=np.int32).reshape(-1, 6),
                   np.asarray(rows, dtype=np.int32), tok)


def build_backward(result: ScheduleResult, lay: RankLayout) -> list[BwdLaunch]:
    deps = result.deps
    causal = deps.mask == CAUSAL
    consumers: dict[ChunkKey, list[ChunkKey]] = {}
    local = set(lay.chunks)
    for q in lay.chunks:
        for kv in deps.q_to_kv[q]:
            consumers.setdefault(kv, []).append(q)
    launches = []
    for recv in (True, False):
        kv_list = lay.recv_chunks if recv else lay.chunks
        kvsegs, qrefs, items, pairs = [], [], [], 0
        kv_keys, q_keys = [], []
        for kv in kv_list:
            qs = consumers.get(kv, [])
            if not qs:
                # a local chunk no local Q attends to, or a chunk this rank only relays
                # (ring / ByteScale plans): no dK/dV work here
                continue
            kn = deps.chunk_tokens[kv]
            off = lay.recv_offset[kv] if recv else lay.offset[kv]
            begin = len(qrefs)
            for q in qs:
                assert q in local
                diag = int(causal and q == kv)
                qrefs.append((lay.offset[q], deps.chunk_tokens[q], diag, 0))
                q_keys.append(q)
                pairs += tile_token_pairs(deps.chunk_tokens[q], kn, bool(diag))
            kidx = len(kvsegs)
            kvsegs.append((off, kn, KV_RECV if recv else 0, begin, len(qrefs), 0))
            kv_keys.append(kv)
            for nb in range(_cdiv(kn, TILE)):
                cost = 0
                for q in qs:
                    qb = _cdiv(deps.chunk_tokens[q], TILE)
                    cost += qb - nb if (causal and q == kv) else qb
                items.append((cost, kidx, nb, kv[0]))
        if not kvsegs:
            continue
        items = _lpt_order(items)
        launches.append(BwdLaunch(
            recv, np.asarray(kvsegs, dtype=np.int32).reshape(-1, 6),
            np.asarray(qrefs, dtype=np.int32).reshape(-1, 4),
            np.asarray([(k, b) for _, k, b, _ in items], dtype=np.int32).reshape(-1, 2), pairs,
            np.asarray([c for c, _, _, _ in items], dtype=np.int64), kv_keys, q_keys))
    return launches


def build_dq(result: ScheduleResult, lay: RankLayout) -> DqPlan:
    deps = result.deps
    causal = deps.mask == CAUSAL
    segs, refs, items, pairs = [], [], [], 0
    q_keys, kv_keys = [], []
    for q in lay.chunks:
        qn = deps.chunk_tokens[q]
        begin = len(refs)
        q_keys.append(q)
        for kv in deps.q_to_kv[q]:
            kv_keys.append(kv)
            _, off, flags = _kv_location(lay, kv)
            if causal and kv == q:
                flags |= KV_DIAG
            refs.append((off, deps.chunk_tokens[kv], flags, 0))
            pairs += tile_token_pairs(qn, deps.chunk_tokens[kv], bool(flags & KV_DIAG))
        sidx = len(segs)
        segs.append((lay.offset[q], qn, begin, len(refs), -1, 0))
        for mb in range(_cdiv(qn, TILE)):
            cost = 0
            for off, kn, flags, _ in refs[begin:]:
                nt = _cdiv(kn, TILE)
                cost += min(nt, mb + 1) if flags & KV_DIAG else nt
            items.append((cost, sidx, mb, q[0]))
    items = _lpt_order(items)
    return DqPlan(np.asarray(segs, dtype=np.int32).reshape(-1, 6),
                  np.asarray(refs, dtype=np.int32).reshape(-1, 4),
                  np.asarray([(s_, m) for _, s_, m, _ in items], dtype=np.int32).reshape(-1, 2),
                  pairs, np.asarray([c for c, _, _, _ in items], dtype=np.int64), q_keys, kv_keys)


def build_ds_tiles(bwd: list[BwdLaunch], dq: DqPlan, causal: bool) -> int:
    """Materialised-dS backward: number the (KV block, Q block) pairs in the order the
    dK/dV kernel visits them (launch, item in LPT order, qref, q block) -> pair ids.
    Every dK/dV item gets the first id of its pairs (``pair_base``); every dQ item the id
    of each KV tile it visits (``pair_ids``/``pair_off``), so the dQ kernel reads exactly
    the dS tiles the dK/dV kernel wrote: tile = pair * Hq + q head.  Returns the pair
    count."""
    ids: dict = {}
    nxt = 0
    for b in bwd:
        base = []
        for k, nb in b.items.tolist():
            base.append(nxt)
            kv = b.kv_keys[k]
            seg = b.kvsegs[k]
            for r in range(seg[3], seg[4]):
                q_off, q_len, diag, _ = b.qrefs[r].tolist()
                first = nb if diag else 0
                for mb in range(first, _cdiv(q_len, TILE)):
                    ids[(kv, nb, b.q_keys[r], mb)] = nxt
                    nxt += 1
        b.pair_base = np.asarray(base, dtype=np.int32)
    flat, off = [], []
    for s_idx, mb in dq.items.tolist():
        off.append(len(flat))
        seg = dq.segments[s_idx]
        q = dq.q_keys[s_idx]
        for r in range(seg[2], seg[3]):
            kv_off, kv_len, flags, _ = dq.kvrefs[r].tolist()
            nt = _cdiv(kv_len, TILE)
            if flags & KV_DIAG:
                nt = min(nt, mb + 1)
            for t in range(nt):
                flat.append(ids[(dq.kv_keys[r], t, q, mb)])
    dq.pair_ids = np.asarray(flat, dtype=np.int32)
    dq.pair_off = np.asarray(off, dtype=np.int32)
    return nxt


def build_rank_work(result: ScheduleResult, rank: int, fuse_remote: bool = False) -> RankWork:
    lay = rank_layout(result, rank)
    fwd = build_forward(result, lay, fuse_remote)
    bwd = build_backward(result, lay)
    dq = build_dq(result, lay)
    n_pairs = build_ds_tiles(bwd, dq, result.deps.mask == CAUSAL)
    return RankWork(lay, fwd, bwd, sum(w.pairs for w in fwd.waves), dq, n_pairs)
