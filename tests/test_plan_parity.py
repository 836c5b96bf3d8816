"""Control-plane parity: the product planner emits the reference's exact plan.

Golden hashes in ``tests/golden/plan_hashes.json`` were produced by the
unmodified reference planner (``oracle/gen_plan_golden.py``): SURVEY Appendix A
recipes C1-C5 at N=1/2/4/8 plus a 1,200-case seeded corpus (both masks,
coalesce 1/4/16, infeasible batches included).
"""

import json
import os

import pytest

from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, ModelConfig
from paper_2605_08524_b200.pipeline import fcp_schedule, plan_digest
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.workload import Batch, Sequence

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "plan_hashes.json")
CASES = json.load(open(GOLDEN))["cases"]

# SURVEY Appendix A, copied from the survey's table (reference output).
APPENDIX_A = {
    ("C1-tiny", 2): "a43df7a41c9318fd",
    ("C2-llama3-8b-64k", 1): "4ec0b94155a749d2", ("C2-llama3-8b-64k", 2): "5c6aaaf95acc8d21",
    ("C2-llama3-8b-64k", 4): "1bc2f1b9c820ea33", ("C2-llama3-8b-64k", 8): "13571c6744872391",
    ("C3-long-tail", 1): "7e84cffd2e22c712", ("C3-long-tail", 2): "010b1e22dea33191",
    ("C3-long-tail", 4): "0b4c106b0158d011", ("C3-long-tail", 8): "3052eb9b1c1a540f",
    ("C4-uniform-128k", 1): "1c76ebb6eeaaa5f9", ("C4-uniform-128k", 2): "915f0b65fdb9ae41",
    ("C4-uniform-128k", 4): "b926768328b0ce1e", ("C4-uniform-128k", 8): "54771d777d650aee",
    ("C5-b1024", 8): "ac3468a2c582ea13", ("C5-b6144", 8): "9d4afa607f47e72e",
}


def _run(case):
    model = ModelConfig(**case["model"])
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(case["lengths"])),
                  case["n"], case["tpw"])
    try:
        r = fcp_schedule(batch, case["n"], ShardingConfig(case["block"], case["mask"]), model,
                         DEFAULT_EFFICIENCY, coalesce_degree=case["coalesce"])
    except Exception as exc:
        return "raise:" + type(exc).__name__
    return plan_digest(r, model)


def test_appendix_a_hashes_recorded():
    seen = {(c["name"], c["n"]): c["sha"] for c in CASES}
    for key, sha in APPENDIX_A.items():
        assert seen[key] == sha, key


@pytest.mark.parametrize("chunk", range(8))
def test_plan_bit_identical(chunk):
    part = CASES[chunk::8]
    bad = [(c["name"], c["sha"], got) for c in part if (got := _run(c)) != c["sha"]]
    assert not bad, bad[:5]


GOLDEN_B200 = os.path.join(os.path.dirname(__file__), "golden", "plan_hashes_b200_curve.json")


def test_plan_bit_identical_with_b200_curve():
    """`bench.py --curve b200` plans: the product planner with costmodel.B200_EFFICIENCY
    against the unmodified reference run with the same anchors (oracle/gen_plan_golden_b200.py)."""
    from paper_2605_08524_b200 import configs
    from paper_2605_08524_b200.costmodel import B200_EFFICIENCY
    g = json.load(open(GOLDEN_B200))
    assert [list(a) for a in B200_EFFICIENCY.anchors] == g["curve_anchors"], \
        "B200_EFFICIENCY changed: rerun oracle/gen_plan_golden_b200.py"
    by_name = {"C2-llama3-8b-64k": lambda n, b: configs.c2_llama8b_64k(n),
               "C3-long-tail": lambda n, b: configs.c3_long_tail(n),
               "C4-uniform-128k": lambda n, b: configs.c4_uniform_128k(n)}
    bad = []
    for c in g["cases"]:
        make = by_name.get(c["name"], lambda n, b: configs.c5_block_sweep(n, b))
        w = make(c["n"], c["block"])
        r = fcp_schedule(w.batch(), c["n"], ShardingConfig(block_size=w.block_size), w.model,
                         B200_EFFICIENCY)
        if plan_digest(r, w.model) != c["sha"]:
            bad.append((c["name"], c["n"]))
    assert not bad, bad
