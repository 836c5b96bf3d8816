"""The K5/K6 transport's host logic on CPU: the copy lists the executor issues
(``p2p.stage_pulls``, ``p2p.return_pulls``) against the plan and the reference's arrival
semantics (``simulator.py:112-133``).

* every received chunk is pulled exactly once, from its owner, in the stage the reference
  says it arrives (relay plans included), and the merged runs tile the receive arena;
* every (chunk, consumer) dK/dV partial is pulled back exactly once by the chunk's owner,
  from the consumer's receive-arena rows, and the runs tile the owner's staging rows.
"""

import numpy as np
import pytest

from oracle import reference_plan
from paper_2605_08524_b200 import exchange
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, ModelConfig
from paper_2605_08524_b200.distributor import chunk_placement
from paper_2605_08524_b200.p2p import return_pulls, stage_pulls
from paper_2605_08524_b200.pipeline import fcp_schedule
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.simmodel import arrival_stages
from paper_2605_08524_b200.workload import Batch, Sequence
from paper_2605_08524_b200.worklist import rank_layout

MODEL = ModelConfig(q_heads=32, kv_heads=8, head_dim=128)
MIX = [9000, 5100, 4100, 3000, 2100, 1500, 1000, 700, 513, 300, 129, 128, 127, 40, 5]


def _plan(lengths, n, block, sched="fcp", coalesce=16):
    tpw = -(-sum(lengths) // n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(lengths)), n, tpw)
    if sched == "ring":
        from paper_2605_08524_b200.baselines import ring_schedule
        return ring_schedule(batch, n, MODEL)
    if sched == "bytescale":
        from paper_2605_08524_b200.baselines import bytescale_schedule
        return bytescale_schedule(batch, n, tpw, MODEL)
    return fcp_schedule(batch, n, ShardingConfig(block), MODEL, DEFAULT_EFFICIENCY, coalesce_degree=coalesce)


def _arrivals(result, owner):
    """(chunk, worker) -> arrival stage, from the unmodified reference when present."""
    if reference_plan.available():
        import sys
        ref = reference_plan.load()  # noqa: F841
        return sys.modules[f"{reference_plan.ALIAS}.simulator"]._arrival_stages(result.plan.stages, owner)
    return arrival_stages(result.plan.stages, owner)


CASES = [
    (MIX, 2, 2048, "fcp", 16), (MIX, 3, 1024, "fcp", 16), (MIX, 4, 1024, "fcp", 4),
    (MIX, 8, 512, "fcp", 16), (MIX, 8, 512, "fcp", 1), (MIX, 4, 1024, "ring", 16),
    (MIX, 4, 1024, "bytescale", 16),
]


@pytest.mark.parametrize("lengths,n,block,sched,coalesce", CASES)
def test_forward_pulls_follow_plan(lengths, n, block, sched, coalesce):
    r = _plan(lengths, n, block, sched, coalesce)
    owner = chunk_placement(r.assignment, r.units)
    arrival = _arrivals(r, owner)
    layouts = [rank_layout(r, q) for q in range(n)]
    total_pulled = 0
    for rank, lay in enumerate(layouts):
        pulls = stage_pulls(r, rank, layouts, owner)
        assert len(pulls) == len(r.plan.stages)
        chunk_at = {}
        for c in lay.recv_chunks:
            for i in range(lay.chunk_tokens[c]):
                chunk_at[lay.recv_offset[c] + i] = c
        cover = np.zeros(lay.recv_tokens, dtype=np.int64)
        for s, stage in enumerate(pulls):
            chunks_this_stage = set()
            for p in stage:
                assert p.peer != rank and p.rows > 0
                cover[p.dst:p.dst + p.rows] += 1
                row = p.dst
                while row < p.dst + p.rows:                 # walk the chunks of a merged run
                    c = chunk_at[row]
                    assert lay.recv_offset[c] == row, "runs start and end on chunk boundaries"
                    assert owner[c] == p.peer, "pulled from the owner"
                    assert layouts[p.peer].offset[c] == p.src + (row - p.dst), "source rows"
                    assert arrival[(c, rank)] == s == lay.recv_stage[c], "pulled in its arrival stage"
                    chunks_this_stage.add(c)
                    row += lay.chunk_tokens[c]
                assert row == p.dst + p.rows
            if sched == "fcp":
                # a coalesced stage is <= degree matchings: <= degree chunks into each GPU
                assert len(chunks_this_stage) <= r.plan.degree
        assert (cover == 1).all(), "the runs tile the receive arena exactly once"
        total_pulled += lay.recv_tokens
    # every (chunk, destination) the plan delivers is pulled by that destination
    delivered = {(c, e.dst) for st in r.plan.stages for e in st for c in e.chunks}
    assert sum(layouts[d].chunk_tokens[c] for c, d in delivered) == total_pulled


@pytest.mark.parametrize("lengths,n,block,sched,coalesce", CASES)
def test_return_pulls_bring_every_partial_home(lengths, n, block, sched, coalesce):
    r = _plan(lengths, n, block, sched, coalesce)
    owner = chunk_placement(r.assignment, r.units)
    layouts = [rank_layout(r, q) for q in range(n)]
    consumer_cover = [np.zeros(l.recv_tokens, dtype=np.int64) for l in layouts]
    for rank in range(n):
        returns = exchange.owner_returns(layouts, owner, rank)
        rows, rounds, total = exchange.return_staging_layout(returns)
        pulls = return_pulls(returns, layouts, rows)
        want = {(c, q) for q, l in enumerate(layouts) if q != rank
                for c in l.recv_chunks if c in l.consumed and owner[c] == rank}
        assert {(t.chunk, t.peer) for t in returns} == want
        staged = np.zeros(total, dtype=np.int64)
        by_row = {rows[(t.chunk, t.peer)]: t for t in returns}
        for p in pulls:
            staged[p.dst:p.dst + p.rows] += 1
            row = p.dst
            while row < p.dst + p.rows:
                t = by_row[row]
                assert t.peer == p.peer
                assert layouts[t.peer].recv_offset[t.chunk] == p.src + (row - p.dst)
                consumer_cover[t.peer][layouts[t.peer].recv_offset[t.chunk]:
                                       layouts[t.peer].recv_offset[t.chunk] + t.tokens] += 1
                row += t.tokens
            assert row == p.dst + p.rows
        assert (staged == 1).all(), "the runs tile the staging rows exactly once"
        # K4's CSR: every staged row feeds exactly one of my local rows
        assert sorted(x for src, _ in rounds for x in src) == list(range(total))
    for q, l in enumerate(layouts):
        for c in l.recv_chunks:
            a, m = l.recv_offset[c], l.chunk_tokens[c]
            # consumed partials go home once; relay-only chunks have no partial to return
            assert (consumer_cover[q][a:a + m] == (1 if c in l.consumed else 0)).all(), (q, c)


def test_c2_and_c3_plans_at_eight_ranks():
    """The bench workloads' plans (Appendix A recipes): C2 and C3 at N=8."""
    from paper_2605_08524_b200 import configs
    for name in ("c2", "c3"):
        w = configs.by_name(name, 8)
        r = fcp_schedule(w.batch(), 8, ShardingConfig(w.block_size), w.model, DEFAULT_EFFICIENCY)
        owner = chunk_placement(r.assignment, r.units)
        layouts = [rank_layout(r, q) for q in range(8)]
        for rank, lay in enumerate(layouts):
            cover = np.zeros(lay.recv_tokens, dtype=np.int64)
            for stage in stage_pulls(r, rank, layouts, owner):
                for p in stage:
                    cover[p.dst:p.dst + p.rows] += 1
            assert (cover == 1).all()
