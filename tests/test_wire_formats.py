"""precomputed schedule/plan wire formats (blocksched.schedule/1,
blocksched.plan/1; reference cli.py:214-258) consumed directly.  Round trip through our
own payloads, and -- where /root/reference exists -- through the reference CLI's
serialisers, must give the identical plan (digest) and identical device work lists."""

import json

import numpy as np
import pytest

from oracle import reference_plan
from paper_2605_08524_b200 import configs
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY
from paper_2605_08524_b200.errors import ParameterError
from paper_2605_08524_b200.pipeline import (fcp_schedule, plan_digest, plan_payload,
                                            result_from_payloads, schedule_payload)
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.workload import Batch, Sequence
from paper_2605_08524_b200.worklist import build_rank_work


def _plan(name, n):
    w = configs.by_name(name, n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(w.lengths)), n, w.tokens_per_worker)
    return w, fcp_schedule(batch, n, ShardingConfig(w.block_size), w.model, DEFAULT_EFFICIENCY)


def _same_work(a, b, n):
    for r in range(n):
        wa, wb = build_rank_work(a, r), build_rank_work(b, r)
        assert wa.layout.offset == wb.layout.offset and wa.layout.recv_offset == wb.layout.recv_offset
        for xa, xb in zip(wa.fwd.waves, wb.fwd.waves):
            assert np.array_equal(xa.segments, xb.segments) and np.array_equal(xa.items, xb.items)


@pytest.mark.parametrize("name,n", [("c1", 2), ("c2", 4), ("c2", 8)])
def test_own_payload_round_trip(name, n):
    w, r = _plan(name, n)
    sched = json.loads(json.dumps(schedule_payload(r, w.model)))     # through JSON text
    pl = json.loads(json.dumps(plan_payload(r.sub_stage_plan, r.plan.degree)))
    back = result_from_payloads(sched, pl)
    assert plan_digest(back, w.model) == plan_digest(r, w.model)
    _same_work(r, back, n)


@pytest.mark.skipif(not reference_plan.available(), reason="reference package not present")
@pytest.mark.parametrize("name,n", [("c2", 4), ("c3", 2)])
def test_reference_cli_payloads(name, n):
    """The reference CLI's own serialisers (cli.schedule_payload / plan_payload) applied to
    the reference's own fcp_schedule -> our executor's work lists."""
    import sys
    w, ours = _plan(name, n)
    model_kw = dict(q_heads=w.model.q_heads, kv_heads=w.model.kv_heads, head_dim=w.model.head_dim,
                    dtype_bytes=w.model.dtype_bytes)
    h, rr = reference_plan.reference_digest(list(w.lengths), n, w.tokens_per_worker, w.block_size, model_kw)
    cli = sys.modules[f"{reference_plan.ALIAS}.cli"]
    ref = reference_plan.load()
    sched = json.loads(json.dumps(cli.schedule_payload(rr, ref.ModelConfig(**model_kw))))
    pl = json.loads(json.dumps(cli.plan_payload(rr.sub_stage_plan, rr.plan.degree)))
    back = result_from_payloads(sched, pl)
    assert plan_digest(back, w.model) == h == plan_digest(ours, w.model)
    _same_work(ours, back, n)


def test_bad_payloads():
    w, r = _plan("c1", 2)
    with pytest.raises(ParameterError):
        result_from_payloads({"format": "x"}, plan_payload(r.sub_stage_plan, r.plan.degree))
