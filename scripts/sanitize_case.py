"""Small fwd+bwd cases for compute-sanitizer (memcheck / racecheck / synccheck): C1 lengths at
8/2 heads on 1 and 2 simulated ranks (merge + dKV return), both dQ modes, and one C2-shape
sequence set at 32/8 heads.  Exits non-zero if the results leave the stated tolerance.

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.simworkers import global_offsets  # noqa: E402
from paper_2605_08524_b200 import configs  # noqa: E402
from paper_2605_08524_b200.costmodel import ModelConfig  # noqa: E402
from tests.gpu_harness import (assert_within_tolerance, compare, make_inputs, oracle,  # noqa: E402
                               run_plan_on_gpu, schedule)


def case(lengths, n, block, model):
    r = schedule(lengths, n, block, model)
    _, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    gpu = run_plan_on_gpu(r, model, q, k, v, do)
    torch.cuda.synchronize()
    ref, idx = oracle(r, model, q, k, v, do)
    rep = compare(gpu, ref, idx)
    assert_within_tolerance(rep)
    print("ok", n, block, len(lengths), {k_: round(e["rel_l2"], 5) for k_, e in rep.items()}, flush=True)


def main():
    small = ModelConfig(q_heads=8, kv_heads=2, head_dim=128)
    c1 = list(configs.c1_tiny(2).lengths)
    case(c1, 1, 512, small)
    case(c1, 2, 512, small)
    os.environ["FCPB_DS"] = "0"
    case(c1, 2, 512, small)
    del os.environ["FCPB_DS"]
    case([3000, 1200, 700, 129], 1, 2048, configs.LLAMA3_8B)


if __name__ == "__main__":
    main()
