"""the reference's competitor schedulers (``baselines.py:17-181``), so their
plans run on the same B200 executor as FCP's.

* ``ring_schedule`` (``baselines.py:75-99``): every sequence is cut into 2N chunks, rank k
  holds the zigzag pair (k, 2N-1-k), and the KV bundles rotate one neighbour per round for
  N-1 rounds (``_ring_rounds``, ``baselines.py:41-72``).
* ``bytescale_schedule`` (``baselines.py:107-158``): a sequence of length L gets a
  power-of-two group of ceil(L / tokens_per_worker) ranks.  Groups are placed first-fit on
  aligned windows with token capacity left, falling back to the least-overloaded window,
  and each group runs its own ring.
* ``wlb_oracle`` (``baselines.py:161-181``): simulate both, keep the faster.

Relay edges (a rank forwarding a bundle it received) only say *when* a chunk reaches a
rank.  On NVSwitch the executor pulls every chunk straight from its owner's symmetric
buffer, and returns dK/dV partials to the owner from every rank that received the chunk.
"""

from __future__ import annotations

from .costmodel import EfficiencyCurve, HardwareConfig, ModelConfig, kv_chunk_bytes
from .distributor import Assignment
from .errors import InfeasibleError
from .pipeline import ScheduleResult
from .planner import CoalescedPlan, CommPlan, Edge
from .sharding import (CAUSAL, Chunk, ScheduleUnit, ZIGZAG_PAIR, chunk_token_counts,
                       kv_dependencies, zigzag_pairs)
from .simmodel import SimOptions, simulate
from .workload import Batch


def _zigzag_over(seq, workers: list[int], first_unit_id: int):
    """Cut ``seq`` into 2g chunks (g = len(workers)); the member at position k of the group
    gets the pair (k, 2g-1-k).  Returns (units, unit -> worker, worker -> its chunks)."""
    g = len(workers)
    sizes = chunk_token_counts(seq.length, 2 * g)
    by_index = {i: Chunk(seq.id, i, t) for i, t in enumerate(sizes) if t > 0}
    units, where = [], {}
    held: dict[int, list[Chunk]] = {w: [] for w in workers}
    for pos, pair in enumerate(zigzag_pairs(g)):
        members = tuple(by_index[i] for i in pair if i in by_index)
        if not members:
            continue
        unit = ScheduleUnit(first_unit_id + len(units), ZIGZAG_PAIR, members)
        units.append(unit)
        where[unit.unit_id] = workers[pos]
        held[workers[pos]].extend(members)
    return units, where, held


def _rotations(groups, cfg: ModelConfig) -> list[list[Edge]]:
    """Round r of a size-g group (r < g-1): position k forwards the bundle that started at
    position k-r (mod g) to position k+1 (mod g).  Same-round bundles on one (src, dst)
    become one edge; edges are ordered by (src, dst)."""
    rounds = []
    longest = max((len(members) for members, _ in groups), default=0)
    for r in range(max(longest - 1, 0)):
        moving: dict[tuple[int, int], list[Chunk]] = {}
        for members, held in groups:
            g = len(members)
            if r >= g - 1:
                continue
            for pos, w in enumerate(members):
                bundle = held[members[(pos - r) % g]]
                if bundle:
                    moving.setdefault((w, members[(pos + 1) % g]), []).extend(bundle)
        edges = [Edge(src, dst, tuple(c.key for c in moving[(src, dst)]),
                      sum(kv_chunk_bytes(c.token_count, cfg) for c in moving[(src, dst)]))
                 for src, dst in sorted(moving)]
        if edges:
            rounds.append(edges)
    return rounds


def _result(label, units, where, groups, n, cfg, mask) -> ScheduleResult:
    memory = [0.0] * n
    for u in units:
        memory[where[u.unit_id]] += u.token_count
    rounds = _rotations(groups, cfg)
    # round r forwards what arrived in round r-1: never coalesce (degree 1)
    return ScheduleResult(label, units, kv_dependencies(units, mask),
                          Assignment(n, dict(where), memory, [0.0] * n), CommPlan(n, rounds),
                          CoalescedPlan(n, 1, [list(rnd) for rnd in rounds]))


def ring_schedule(batch: Batch, n_workers: int, cfg: ModelConfig, mask: str = CAUSAL) -> ScheduleResult:
    """Monolithic ring over all ranks for every sequence."""
    everyone = list(range(n_workers))
    units, where = [], {}
    held: dict[int, list[Chunk]] = {w: [] for w in everyone}
    for seq in batch.sequences:
        su, sw, sh = _zigzag_over(seq, everyone, len(units))
        units += su
        where.update(sw)
        for w, chunks in sh.items():
            held[w] += chunks
    return _result("ring", units, where, [(everyone, held)], n_workers, cfg, mask)


def _group_size(length: int, tokens_per_worker: int) -> int:
    need = max(1, -(-length // tokens_per_worker))
    return 1 << (need - 1).bit_length()


def bytescale_schedule(batch: Batch, n_workers: int, tokens_per_worker: int,
                       cfg: ModelConfig, mask: str = CAUSAL) -> ScheduleResult:
    """Length-proportional power-of-two groups, each running its own ring."""
    seqs = sorted(batch.sequences,
                  key=lambda s: (-_group_size(s.length, tokens_per_worker), -s.length, s.id))
    room = [float(tokens_per_worker)] * n_workers
    units, where, groups = [], {}, []
    for seq in seqs:
        g = _group_size(seq.length, tokens_per_worker)
        if g > n_workers:
            raise InfeasibleError(
                f"sequence {seq.id} needs a group of {g} workers, cluster has {n_workers}")
        sizes = chunk_token_counts(seq.length, 2 * g)
        need = [sizes[k] + sizes[2 * g - 1 - k] for k in range(g)]
        starts = range(0, n_workers - g + 1, g)
        fit = [s for s in starts if all(room[s + k] >= need[k] for k in range(g))]
        start = fit[0] if fit else min(starts, key=lambda s: max(need[k] - room[s + k] for k in range(g)))
        members = list(range(start, start + g))
        su, sw, sh = _zigzag_over(seq, members, len(units))
        units += su
        where.update(sw)
        groups.append((members, sh))
        for k, w in enumerate(members):
            room[w] -= need[k]
    return _result("bytescale", units, where, groups, n_workers, cfg, mask)


def wlb_oracle(batch: Batch, n_workers: int, tokens_per_worker: int, hw: HardwareConfig,
               cfg: ModelConfig, curve: EfficiencyCurve, opts: SimOptions | None = None,
               mask: str = CAUSAL) -> tuple[ScheduleResult, str]:
    """Simulate ring and (if feasible) the grouped scheduler; keep whichever finishes first
    (ring on ties)."""
    opts = opts or SimOptions()

    def sim_time(res):
        return simulate(res.assignment, res.plan, res.units, res.deps, hw, cfg, curve, opts).total_time

    best = ring_schedule(batch, n_workers, cfg, mask)
    best_t = sim_time(best)
    try:
        grouped = bytescale_schedule(batch, n_workers, tokens_per_worker, cfg, mask)
    except InfeasibleError:
        grouped = None
    if grouped is not None:
        t = sim_time(grouped)
        if t < best_t:
            best, best_t = grouped, t
    return best, best.label
