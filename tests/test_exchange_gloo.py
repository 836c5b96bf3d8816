"""Multi-process exchange on CPU (gloo, world_size 2 and 3, 127.0.0.1).

Executes the product transport's copy lists -- ``p2p.stage_pulls`` per coalesced stage and
``p2p.return_pulls`` for the reversed-edge dK/dV return, each run moving two planes (K and
V, dK and dV) exactly as the executor's 2-D copy-engine pulls do -- with real
point-to-point messages between processes: a pull (peer, src, dst, rows) becomes a message
the peer serves from its own plane rows [src, src+rows).  Checks that (a) every rank's
two-plane receive arena ends up holding exactly the K/V rows of the chunks the plan delivers
to it and (b) the return brings every consumer's partial back to the owner's staging rows.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.simworkers import gather_rank, global_offsets
from paper_2605_08524_b200 import exchange
from paper_2605_08524_b200.p2p import return_pulls, stage_pulls
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, ModelConfig
from paper_2605_08524_b200.pipeline import fcp_schedule, plan_digest
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.workload import Batch, Sequence
from paper_2605_08524_b200.distributor import chunk_placement
from paper_2605_08524_b200.worklist import rank_layout

MODEL = ModelConfig(q_heads=4, kv_heads=2, head_dim=8)
LENGTHS = [3000, 1700, 900, 400, 130, 77, 5]


def _schedule(n, sched="fcp"):
    tpw = -(-sum(LENGTHS) // n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(LENGTHS)), n, tpw)
    if sched == "ring":
        from paper_2605_08524_b200.baselines import ring_schedule
        return ring_schedule(batch, n, MODEL)
    return fcp_schedule(batch, n, ShardingConfig(256), MODEL, DEFAULT_EFFICIENCY, coalesce_degree=4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _serve_and_pull(rank, world, pulls_of, s, src_planes, dst_planes):
    """One stage of pulls as gloo messages: serve every peer's pulls from my planes, receive
    mine into ``dst_planes``; both sides walk the same lists in the same order."""
    ops, landing = [], []
    for q in range(world):
        if q == rank:
            continue
        for p in pulls_of[q][s]:
            if p.peer == rank:
                ops.append(dist.P2POp(dist.isend, src_planes[:, p.src:p.src + p.rows].contiguous(), q))
    for p in pulls_of[rank][s]:
        buf = torch.empty_like(dst_planes[:, p.dst:p.dst + p.rows])
        ops.append(dist.P2POp(dist.irecv, buf, p.peer))
        landing.append((p, buf))
    for w in (dist.batch_isend_irecv(ops) if ops else []):
        w.wait()
    for p, buf in landing:
        dst_planes[:, p.dst:p.dst + p.rows] = buf


def _worker(rank, world, port, errq, sched="fcp"):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        r = _schedule(world, sched)
        exchange.sync_plan_digest(plan_digest(r, MODEL))
        lay = rank_layout(r, rank)
        goff, T = global_offsets(r)
        g = torch.Generator().manual_seed(7)
        kg = torch.randn((T, MODEL.kv_heads, MODEL.head_dim), generator=g)
        vg = torch.randn((T, MODEL.kv_heads, MODEL.head_dim), generator=g)
        k = gather_rank(kg, lay, goff, r.deps)
        v = gather_rank(vg, lay, goff, r.deps)
        layouts = [rank_layout(r, q) for q in range(world)]
        owner = chunk_placement(r.assignment, r.units)
        kv = torch.stack([k, v])                                # my two planes
        kv_recv = torch.full((2, lay.recv_tokens, MODEL.kv_heads, MODEL.head_dim), float("nan"))
        pulls_of = [stage_pulls(r, q, layouts, owner) for q in range(world)]
        for s_idx in range(len(r.plan.stages)):
            _serve_and_pull(rank, world, pulls_of, s_idx, kv, kv_recv)
        assert torch.equal(kv_recv[0], gather_rank(kg, lay, goff, r.deps, recv=True))
        assert torch.equal(kv_recv[1], gather_rank(vg, lay, goff, r.deps, recv=True))
        # reverse: each consumer's "partial" = (its rank + chunk data); owners pull them home
        part = kv_recv + 1000.0 * (rank + 1)
        rets = [exchange.owner_returns(layouts, owner, q) for q in range(world)]
        staging = [exchange.return_staging_layout(t) for t in rets]
        rpulls = [[return_pulls(rets[q], layouts, staging[q][0])] for q in range(world)]
        rows, rounds, n_stage = staging[rank]
        staged = torch.zeros((2, n_stage, MODEL.kv_heads, MODEL.head_dim))
        _serve_and_pull(rank, world, rpulls, 0, part, staged)
        for t in rets[rank]:
            a_ = rows[(t.chunk, t.peer)]
            want = kv[:, t.row:t.row + t.tokens] + 1000.0 * (t.peer + 1)
            assert torch.equal(staged[:, a_:a_ + t.tokens], want), (rank, t)
        # rounds: every staged row used once; destinations unique within a round
        srcs = sorted(x for src, _ in rounds for x in src)
        assert srcs == list(range(n_stage))
        for _, dst in rounds:
            assert len(dst) == len(set(dst))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # surface the failure in the parent
        import traceback
        errq.put(f"rank {rank}: {exc!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,sched", [(2, "fcp"), (3, "fcp"), (3, "ring")])
def test_plan_exchange_over_gloo(world, sched):
    r = _schedule(world, sched)
    assert sum(len(s) for s in r.plan.stages) > 0
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, errq, sched)) for i in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
