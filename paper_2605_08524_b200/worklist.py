"""H1: turn a ``ScheduleResult`` into per-rank device work lists.

Nothing here exists in the reference: it is the bridge from the plan the
reference computes (``pipeline.py:31-60``) to the tiles its simulator only
times (``simulator.py:73-109``).  For rank ``r``:

* **Layout.**  Local chunks are packed token-major sorted by (sequence, chunk
  index); this is the layout of the rank's Q, K, V, O, dO, dQ, dK, dV.  Remote
  chunks the rank receives get slots in a *receive arena*, ordered by the
  coalesced stage that delivers them, then by plan edge order
  (``simulator.py:112-133`` defines the arrival stage).
* **Runs.**  Consecutive chunks of one sequence held by the rank are one
  contiguous *run*; a run is executed as one causal segment (its own diagonal
  plus fully visible earlier sources), which computes exactly the tiles of its
  chunks' ``q_to_kv`` lists with raggedness only at the run's end (checked
  against ``q_to_kv`` per member chunk; otherwise one run per chunk).  At N=1
  every sequence is one run.
* **Forward waves.**  Wave -1 holds every (Q run, KV source) tile whose KV is
  local -- the dependency-free prologue; wave s holds tiles whose KV arrives
  with coalesced stage s.  A Q run whose tiles span several waves writes one
  fp32 partial (O, LSE) per wave, merged by K3 afterwards; a Q run served by
  a single wave writes its final bf16 O directly.
* **Received groups.**  Received chunks of one sequence that sit back to back in
  the arena form one KV source (``RecvGroup``); each consumer Q run sees a prefix
  of it (``_group_received``).  A zigzag plan often has a rank receive every other
  chunk of a long sequence, so this removes a ragged KV tile per chunk: C2 at N=2
  computes 8,305 / 8,533 forward / backward tiles on rank 0 instead of 8,777 / 8,785.
  The forward also sorts each Q run's refs by (buffer, offset) so that adjacent
  ranges coalesce (``_merge_refs``).
* **Backward.**  dK/dV work is keyed by KV source (received group or local run):
  the KV block iterates over every local Q run attending to it (with its visible
  prefix, ``FcpbBwdQRef.kv_limit``).  Received groups form their own launch so
  their dK/dV partials can travel back along the reversed plan edges while the
  local runs compute.  dQ is query-stationary: one segment per local Q run over
  all of its (by then resident) KV sources.

Work items are sorted longest-first (LPT over the persistent grid).  Visible-pair
accounting stays the reference's per-chunk ``tile_token_pairs``.
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
PRE_WAVE = -2        # local tiles whose data is already in place before a reshuffle completes


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
    qrefs: np.ndarray            # int32 [Q, 4]: q_off q_len diag kv_limit (0: all KV rows)
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
    """The rank's packed layout: its chunks sorted by (sequence, chunk index), so the
    consecutive chunks of one sequence that the plan places here are adjacent in memory in
    token order (``local_runs``); the receive arena in arrival-stage, then (sequence, chunk) order."""
    n = result.assignment.n_workers
    if not 0 <= rank < n:
        raise ParameterError(f"rank {rank} outside [0, {n})")
    chunks: list[ChunkKey] = []
    sizes = dict(result.deps.chunk_tokens)
    for u in sorted(result.units, key=lambda u: u.unit_id):
        if result.assignment.worker_of(u.unit_id) == rank:
            chunks += [c.key for c in u.members]
    chunks.sort()
    offset, pos = {}, 0
    for c in chunks:
        offset[c] = pos
        pos += sizes[c]
    where = chunk_placement(result.assignment, result.units)
    arrival = arrival_stages(result.plan.stages, where)
    recv = []
    for s, stage in enumerate(result.plan.stages):
        got = sorted({c for e in stage if e.dst == rank for c in e.chunks if arrival[(c, rank)] == s})
        # within a stage in (sequence, chunk) order: consecutive chunks of a sequence land in
        # consecutive arena rows (one KV ref in the forward) and are pulled as one run from
        # the owner, whose layout holds them in the same order
        recv += [c for c in got if c not in recv]
    roff, rpos = {}, 0
    for c in recv:
        roff[c] = rpos
        rpos += sizes[c]
    rstage = {c: arrival[(c, rank)] for c in recv}
    needed = {kv for q in chunks for kv in result.deps.q_to_kv[q]}
    return RankLayout(rank, chunks, offset, pos, recv, roff, rpos, rstage, sizes,
                      frozenset(c for c in recv if c in needed))


@dataclass(frozen=True)
class Run:
    """Consecutive chunks ``first..last`` of sequence ``seq`` held by this rank, adjacent in
    its layout: one contiguous token range [off, off + tokens) in sequence order."""
    seq: int
    first: int
    last: int
    off: int
    tokens: int

    @property
    def key(self):
        return ("run", self.seq, self.first, self.last)

    def chunks(self):
        return [(self.seq, i) for i in range(self.first, self.last + 1)]


@dataclass(frozen=True)
class RecvGroup:
    """Received chunks ``chunks`` (one sequence) that sit back to back in the receive arena,
    arrive in the same stage and have the same consumer Q runs: one KV source of
    [off, off + tokens) arena rows, so the forward, dK/dV and dQ tables tile it as one range
    (a ragged tile only at its end, not at every chunk boundary)."""
    chunks_: tuple
    off: int
    tokens: int

    @property
    def key(self):
        return ("recv", self.chunks_[0][0], self.chunks_[0][1], self.chunks_[-1][1])

    def chunks(self):
        return list(self.chunks_)


def local_runs(result: ScheduleResult, lay: RankLayout, merge: bool = True) -> list[Run]:
    """Maximal runs of a rank's chunks (``merge=False``: one run per chunk).  The tile
    geometry of the reference is per chunk (``kv_dependencies``, ``sharding.py:172-201``), and
    a chunk of, say, 920 tokens pads to 8 x 128 rows; a run of consecutive chunks is one
    causal range, so only its end is ragged.  At N=1 every sequence is one run, which on C2
    cuts the 128x128 tiles computed from 17,688 to 14,836 (visible/computed 81% -> 97%).
    Every run's dependency structure is checked against ``q_to_kv`` (``_run_sources``)."""
    runs: list[Run] = []
    for c in lay.chunks:
        n = lay.chunk_tokens[c]
        last = runs[-1] if runs else None
        if (merge and last is not None and last.seq == c[0] and last.last + 1 == c[1]
                and last.off + last.tokens == lay.offset[c]):
            runs[-1] = Run(last.seq, last.first, c[1], last.off, last.tokens + n)
        else:
            runs.append(Run(c[0], c[1], c[1], lay.offset[c], n))
    return runs


def _run_sources(result: ScheduleResult, lay: RankLayout, runs: list[Run]):
    """Per Q run, the KV sources its rows attend to: ("run", S, diag) for local runs (whole
    runs only) and ("recv", chunk) for received chunks, in first-appearance order of the
    members' ``q_to_kv`` lists.  Returns None if any member's visible set is not exactly
    what the run segment encodes: every source fully visible, except the run itself, which
    is causal at row level (chunk p sees chunks a..p-1 fully and itself inclusive-causally,
    ``costmodel.py:141-149``) -- the caller then falls back to one run per chunk."""
    deps = result.deps
    causal = deps.mask == CAUSAL
    run_of = {c: R for R in runs for c in R.chunks()}
    out = {}
    for R in runs:
        members = R.chunks()
        kv_all: list[ChunkKey] = []
        seen = set()
        for p in members:
            for kv in deps.q_to_kv[p]:
                if kv not in seen:
                    seen.add(kv)
                    kv_all.append(kv)
        for p in members:
            want = set(deps.q_to_kv[p])
            got = set(kv_all)
            if causal:
                got -= {c for c in members if c[1] > p[1]}
            if got != want:
                return None
        srcs, taken = [], set()
        for kv in kv_all:
            S = run_of.get(kv)
            if S is None:
                if kv not in lay.recv_offset:
                    raise ConsistencyError(f"plan never delivers chunk {kv} to rank {lay.rank}")
                srcs.append(("recv", kv))
            elif S.key not in taken:
                if not all(c in seen for c in S.chunks()):
                    return None
                taken.add(S.key)
                srcs.append(("run", S, causal and S == R))
        out[R.key] = srcs
    return out


def _group_received(lay: RankLayout, srcs: dict, merge: bool = True, stage_split: bool = False) -> dict:
    """Replace the ("recv", chunk) sources by ("recv", RecvGroup, visible tokens): maximal
    sets of received chunks of one sequence, back to back in the arena in increasing chunk
    order (``merge=False``: one group per chunk; ``stage_split``: and of one arrival stage,
    for per-stage forward waves).  Every Q run that attends to a group sees a *prefix* of it
    (causal: the chunks before the run), so a group is one KV range whose consumers carry
    their visible length -- the dK/dV kernel masks the rows past it (``FcpbBwdQRef.kv_limit``),
    the query-stationary kernels take it as the ref length.  Where a chunk-zigzag plan has a
    rank receive every other chunk of a sequence, this turns per-chunk ragged tiles (a
    920-token chunk computes 8 x 128 rows) into one ragged tile per group.  A candidate group
    whose consumers do not each see a prefix is split into single chunks."""
    consumers: dict = {}
    for q, lst in srcs.items():
        for src in lst:
            if src[0] == "recv":
                consumers.setdefault(src[1], set()).add(q)
    cands, cur = [], None
    for c in lay.recv_chunks:
        if c not in consumers:
            continue
        prev = cur[-1] if cur else None
        if (merge and prev is not None and prev[0] == c[0] and prev[1] < c[1]
                and lay.recv_offset[prev] + lay.chunk_tokens[prev] == lay.recv_offset[c]
                and (not stage_split or lay.recv_stage[prev] == lay.recv_stage[c])):
            cur.append(c)
        else:
            cur = [c]
            cands.append(cur)
    group_of = {}
    for cand in cands:
        # prefix property: the consumer sets shrink along the group
        ok = all(consumers[cand[i + 1]] <= consumers[cand[i]] for i in range(len(cand) - 1))
        for part in ([cand] if ok else [[c] for c in cand]):
            G = RecvGroup(tuple(part), lay.recv_offset[part[0]], sum(lay.chunk_tokens[c] for c in part))
            for c in part:
                group_of[c] = G
    out = {}
    for q, lst in srcs.items():
        new, at = [], {}
        for src in lst:
            if src[0] == "recv":
                G = group_of[src[1]]
                vis = sum(lay.chunk_tokens[c] for c in G.chunks_ if q in consumers[c])
                if G.key in at:
                    continue
                at[G.key] = len(new)
                src = ("recv", G, vis)
            new.append(src)
        out[q] = new
    return out


def _runs_and_sources(result: ScheduleResult, lay: RankLayout, stage_split: bool = False):
    import os
    merge = os.environ.get("FCPB_RUNS", "1") != "0"     # A/B knob: 0 = one segment per chunk
    runs = local_runs(result, lay, merge)
    srcs = _run_sources(result, lay, runs)
    if srcs is None:
        runs = local_runs(result, lay, merge=False)
        srcs = _run_sources(result, lay, runs)
    groups = merge and os.environ.get("FCPB_RECV_GROUPS", "1") != "0"   # A/B knob
    return runs, _group_received(lay, srcs, groups, stage_split)


def _run_pairs(result: ScheduleResult, R: Run, keep) -> int:
    """Visible pairs of the run's member chunks' tiles whose KV chunk satisfies keep(kv)
    (the reference's ``tile_token_pairs`` accounting, per chunk tile)."""
    deps = result.deps
    causal = deps.mask == CAUSAL
    return sum(tile_token_pairs(deps.chunk_tokens[p], deps.chunk_tokens[kv], causal and kv == p)
               for p in R.chunks() for kv in deps.q_to_kv[p] if keep(kv))


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


def _ref_cost(refs, mb) -> int:
    cost = 0
    for _, kn, flags, _ in refs:
        nt = _cdiv(kn, TILE)
        cost += min(nt, mb + 1) if flags & KV_DIAG else nt
    return cost


def _merge_refs(refs):
    """Coalesce fully visible refs that continue each other in the same buffer (forward only:
    the backward's KV blocks must stay aligned with its kvsegs)."""
    out = []
    for r in refs:
        if (out and not (r[2] & KV_DIAG) and not (out[-1][2] & KV_DIAG) and out[-1][2] == r[2]
                and out[-1][0] + out[-1][1] == r[0]):
            out[-1] = (out[-1][0], out[-1][1] + r[1], r[2], 0)
        else:
            out.append(r)
    return out


def build_forward(result: ScheduleResult, lay: RankLayout, fuse_remote: bool = False,
                  resident=None) -> FwdPlan:
    """Forward waves over the rank's Q runs.  fuse_remote: every received KV chunk goes into
    one wave released by this rank's last arrival stage (one launch, one tail, and at most a
    local and a remote partial per Q run) instead of one wave per coalesced stage;
    fuse_remote="all": the local tiles join that wave too (no partials, no merge) -- for ranks
    whose exchange is short next to their compute.  fuse_remote="resume": local wave plus one
    fused remote wave, the remote wave *continuing* each Q run from the local wave's fp32
    (O, LSE) partial (``FcpbSegment.in_row``) and writing the final O -- the local tiles hide
    the exchange and no K3 merge runs.
    resident: chunks whose Q/K/V rows are in place before the reshuffle into the FCP layout
    completes (they stay on this rank); tiles of a resident Q run against a resident local run
    form PRE_WAVE, which runs while the reshuffle pulls the other rows."""
    deps = result.deps
    last_stage = max(lay.recv_stage.values(), default=LOCAL_WAVE)
    runs, sources = _runs_and_sources(result, lay, stage_split=not fuse_remote)
    resident = frozenset(resident or ())

    chain = fuse_remote == "resume"

    def wave_of(kv):
        if kv not in lay.recv_offset:
            return last_stage if fuse_remote == "all" else LOCAL_WAVE
        return last_stage if fuse_remote else lay.recv_stage[kv]

    def is_resident(run):
        return all(c in resident for c in run.chunks())

    pre_pairs: set = set()                 # (Q run key, KV chunk) tiles in PRE_WAVE
    # per Q run: wave -> ordered kv refs
    per_q: dict = {}
    for R in runs:
        waves: dict[int, list] = {}
        r_res = is_resident(R)
        for src in sources[R.key]:
            if src[0] == "run":
                S, diag = src[1], src[2]
                w = PRE_WAVE if (r_res and is_resident(S)) else wave_of(S.chunks()[0])
                if w == PRE_WAVE:
                    pre_pairs.update((R.key, c) for c in S.chunks())
                waves.setdefault(w, []).append((S.off, S.tokens, KV_DIAG if diag else 0, 0))
            else:
                G, vis = src[1], src[2]
                waves.setdefault(wave_of(G.chunks_[0]), []).append((G.off, vis, KV_RECV, 0))
        # the order of a Q run's KV refs is free (online softmax); sorted by (buffer, offset)
        # the refs that continue each other in memory become one range (_merge_refs)
        per_q[R.key] = {w: _merge_refs(sorted(r, key=lambda x: (x[2] & KV_RECV, x[0])))
                        for w, r in waves.items()}

    wave_ids = sorted({w for waves in per_q.values() for w in waves})
    part_rows = 0
    partial_of: dict = {}                 # run key -> [(wave, row)]
    seg_rows: dict = {}                   # (run, wave) -> partial rows it writes
    seg_in: dict = {}                     # (run, wave) -> partial rows it continues (chain)
    for R in runs:
        waves = sorted(per_q[R.key])
        if len(waves) > 1:
            for i, w in enumerate(waves):
                if chain and i > 0:
                    seg_in[(R.key, w)] = seg_rows[(R.key, waves[i - 1])]
                if chain and i == len(waves) - 1:
                    continue              # the last wave of a chain writes the final O
                seg_rows[(R.key, w)] = part_rows
                if not chain:
                    partial_of.setdefault(R.key, []).append((w, part_rows))
                part_rows += R.tokens
    out = []
    for w in wave_ids:
        segs, refs, items, pairs = [], [], [], 0
        for R in runs:
            kvs = per_q[R.key].get(w)
            if not kvs:
                continue
            begin = len(refs)
            refs += kvs
            if w == PRE_WAVE:
                pairs += _run_pairs(result, R, lambda kv: (R.key, kv) in pre_pairs)
            else:
                pairs += _run_pairs(result, R, lambda kv: wave_of(kv) == w and (R.key, kv) not in pre_pairs)
            out_row = seg_rows.get((R.key, w), -1)
            in_row = seg_in[(R.key, w)] + 1 if (R.key, w) in seg_in else 0
            sidx = len(segs)
            segs.append((R.off, R.tokens, begin, len(refs), out_row, in_row))
            for mb in range(_cdiv(R.tokens, TILE)):
                items.append((_ref_cost(kvs, mb), sidx, mb, R.seq))
        items = _lpt_order(items)
        out.append(FwdWave(
            w, np.asarray(segs, dtype=np.int32).reshape(-1, 6),
            np.asarray(refs, dtype=np.int32).reshape(-1, 4),
            np.asarray([(s_, m) for _, s_, m, _ in items], dtype=np.int32).reshape(-1, 2), pairs,
            np.asarray([c for c, _, _, _ in items], dtype=np.int64)))
    groups, rows, tok = [], [], 0
    for R in runs:
        if R.key in partial_of:
            begin = len(rows)
            rows += [r for _, r in partial_of[R.key]]
            groups.append((R.off, R.tokens, begin, len(rows), tok, 0))
            tok += R.tokens
    return FwdPlan(out, part_rows, np.asarray(groups, dtype=np.int32).reshape(-1, 6),
                   np.asarray(rows, dtype=np.int32), tok)


def build_backward(result: ScheduleResult, lay: RankLayout) -> list[BwdLaunch]:
    """dK/dV launches keyed by KV source: received chunks (their partials travel back to
    the owners) and local runs; each iterates the local Q runs that attend to it."""
    deps = result.deps
    runs, sources = _runs_and_sources(result, lay)
    consumers: dict = {}                  # kv key -> [(Q run, diag)]
    kv_src: dict = {}                     # kv key -> (off, tokens, recv, chunk-or-run)
    for R in runs:
        for src in sources[R.key]:
            if src[0] == "run":
                S = src[1]
                consumers.setdefault(S.key, []).append((R, src[2], 0))
                kv_src[S.key] = (S.off, S.tokens, False, S)
            else:
                G, vis = src[1], src[2]
                consumers.setdefault(G.key, []).append((R, False, vis if vis < G.tokens else 0))
                kv_src[G.key] = (G.off, G.tokens, True, G)
    launches = []
    for recv in (True, False):
        keys = (sorted((k for k in consumers if k[0] == "recv"), key=lambda k: kv_src[k][0]) if recv
                else [R.key for R in runs if R.key in consumers])
        kvsegs, qrefs, items, pairs = [], [], [], 0
        kv_keys, q_keys = [], []
        for key in keys:
            off, kn, _, what = kv_src[key]
            qs = consumers[key]
            begin = len(qrefs)
            for R, diag, lim in qs:
                qrefs.append((R.off, R.tokens, int(diag), lim))
                q_keys.append(R.key)
                members = set(what.chunks())
                pairs += _run_pairs(result, R, lambda kv: kv in members)
            kidx = len(kvsegs)
            kvsegs.append((off, kn, KV_RECV if recv else 0, begin, len(qrefs), 0))
            kv_keys.append(key)
            for nb in range(_cdiv(kn, TILE)):
                cost = 0
                for R, diag, lim in qs:
                    qb = _cdiv(R.tokens, TILE)
                    if not _qref_sees(lim, nb):
                        continue
                    cost += qb - nb if diag else qb
                if cost == 0:       # the kernel would wait forever for an accumulator
                    raise ConsistencyError(f"KV block {nb} of {key} has no visiting Q block")
                items.append((cost, kidx, nb, key[1]))
        if not kvsegs:
            continue
        items = _lpt_order(items)
        launches.append(BwdLaunch(
            recv, np.asarray(kvsegs, dtype=np.int32).reshape(-1, 6),
            np.asarray(qrefs, dtype=np.int32).reshape(-1, 4),
            np.asarray([(k, b) for _, k, b, _ in items], dtype=np.int32).reshape(-1, 2), pairs,
            np.asarray([c for c, _, _, _ in items], dtype=np.int64), kv_keys, q_keys))
    return launches


def _qref_sees(kv_limit: int, nb: int) -> bool:
    """Does a dK/dV Q reference with visible prefix ``kv_limit`` (0: all rows) reach KV
    block nb?  (``q_end_block`` in attn_bwd_sm100.cuh.)"""
    return kv_limit == 0 or nb * TILE < kv_limit


def build_dq(result: ScheduleResult, lay: RankLayout) -> DqPlan:
    """Query-stationary dQ tables: one segment per local Q run over all of its KV sources,
    segmented exactly like the backward's kvsegs (so materialised dS tiles line up)."""
    deps = result.deps
    runs, sources = _runs_and_sources(result, lay)
    segs, refs, items, pairs = [], [], [], 0
    q_keys, kv_keys = [], []
    for R in runs:
        begin = len(refs)
        q_keys.append(R.key)
        for src in sources[R.key]:
            if src[0] == "run":
                S, diag = src[1], src[2]
                kv_keys.append(S.key)
                refs.append((S.off, S.tokens, KV_DIAG if diag else 0, 0))
            else:
                G, vis = src[1], src[2]
                kv_keys.append(G.key)
                refs.append((G.off, vis, KV_RECV, 0))
        pairs += _run_pairs(result, R, lambda kv: True)
        sidx = len(segs)
        segs.append((R.off, R.tokens, begin, len(refs), -1, 0))
        for mb in range(_cdiv(R.tokens, TILE)):
            items.append((_ref_cost(refs[begin:], mb), sidx, mb, R.seq))
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
                q_off, q_len, diag, lim = b.qrefs[r].tolist()
                if not _qref_sees(lim, nb):
                    continue
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


def build_rank_work(result: ScheduleResult, rank: int, fuse_remote: bool = False,
                    resident=None) -> RankWork:
    lay = rank_layout(result, rank)
    fwd = build_forward(result, lay, fuse_remote, resident)
    bwd = build_backward(result, lay)
    dq = build_dq(result, lay)
    n_pairs = build_ds_tiles(bwd, dq, result.deps.mask == CAUSAL)
    return RankWork(lay, fwd, bwd, sum(w.pairs for w in fwd.waves), dq, n_pairs)
