"""Multi-process exchange on CPU (gloo, world_size 2 and 3, 127.0.0.1).

Executes the coalesced Delta-matching plan stage by stage with real
point-to-point messages and checks that (a) every rank's receive arena ends up
holding exactly the KV rows of the chunks the plan delivers to it and (b) the
reversed-edge return brings every receiver's partial back to the owner's
staging rows.  This is the host logic of K5/K6 that the NCCL path reuses.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.simworkers import gather_rank, global_offsets
from paper_2605_08524_b200 import exchange
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
        kr = torch.full((lay.recv_tokens, MODEL.kv_heads, MODEL.head_dim), float("nan"))
        vr = kr.clone()
        stages = exchange.build_stage_ops(r, lay)
        for st in stages:
            exchange.wait_all(exchange.run_stage(st, (k, v), (kr, vr)))
        assert torch.equal(kr, gather_rank(kg, lay, goff, r.deps, recv=True))
        assert torch.equal(vr, gather_rank(vg, lay, goff, r.deps, recv=True))
        # reverse: each consumer returns (its rank + chunk data) as the "partial", to the owner
        part = kr + 1000.0 * (rank + 1)
        layouts = [rank_layout(r, q) for q in range(world)]
        owner = chunk_placement(r.assignment, r.units)
        returns = exchange.owner_returns(layouts, owner, rank)
        rows, rounds, n_stage = exchange.return_staging_layout(returns)
        staged = torch.zeros((n_stage, MODEL.kv_heads, MODEL.head_dim))
        exchange.wait_all(exchange.run_return(lay, layouts, owner, (part,), (staged,), rows))
        for t in returns:
            got = staged[rows[(t.chunk, t.peer)]:rows[(t.chunk, t.peer)] + t.tokens]
            want = k[t.row:t.row + t.tokens] + 1000.0 * (t.peer + 1)
            assert torch.equal(got, want), (rank, t)
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
