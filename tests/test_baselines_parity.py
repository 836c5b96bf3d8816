"""ring / ByteScale plans equal the reference's (baselines.py) byte for byte
(canonical schedule+plan digest) on the Appendix A batches; skipped without the reference."""

import hashlib
import json
import sys

import pytest

from oracle import reference_plan
from paper_2605_08524_b200 import configs
from paper_2605_08524_b200.baselines import bytescale_schedule, ring_schedule
from paper_2605_08524_b200.pipeline import plan_digest
from paper_2605_08524_b200.workload import Batch, Sequence

pytestmark = pytest.mark.skipif(not reference_plan.available(), reason="reference package not present")


def _ref_digest(res, model):
    cli = sys.modules[f"{reference_plan.ALIAS}.cli"]
    blob = json.dumps([cli.schedule_payload(res, model),
                       cli.plan_payload(res.sub_stage_plan, res.plan.degree)], sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()[:16]


@pytest.mark.parametrize("name,n", [("c2", 2), ("c2", 4), ("c2", 8), ("c3", 4), ("c5", 8)])
def test_ring_and_bytescale_match_reference(name, n):
    ref = reference_plan.load()
    import importlib
    rb = importlib.import_module(f"{reference_plan.ALIAS}.baselines")
    w = configs.by_name(name, n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(w.lengths)), n, w.tokens_per_worker)
    rbatch = ref.Batch(tuple(ref.Sequence(i, l) for i, l in enumerate(w.lengths)), n, w.tokens_per_worker)
    rm = ref.ModelConfig(w.model.q_heads, w.model.kv_heads, w.model.head_dim, w.model.dtype_bytes)
    assert plan_digest(ring_schedule(batch, n, w.model), w.model) == \
        _ref_digest(rb.ring_schedule(rbatch, n, rm), rm)
    try:
        ref_bs = rb.bytescale_schedule(rbatch, n, w.tokens_per_worker, rm)
    except Exception as exc:     # infeasible there -> must be infeasible here too
        with pytest.raises(type(exc).__name__ and Exception):
            bytescale_schedule(batch, n, w.tokens_per_worker, w.model)
        return
    assert plan_digest(bytescale_schedule(batch, n, w.tokens_per_worker, w.model), w.model) == \
        _ref_digest(ref_bs, rm)
