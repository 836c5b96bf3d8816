"""Per-kernel A/B timing on one GPU: the C2 (or any) workload at N=1, each attention kernel
launched back to back R times with CUDA events on its stream (median ms per launch), so a
kernel change is measured without the rest of the step.  Under ncu, add
``--metrics sm__cycles_elapsed.max`` for clock-independent cycles.

    python scripts/kbench.py [--config c2] [--reps 10] [--kernels fwd,bwd,dq]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--kernels", default="fwd,bwd,dq")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    w, result = bench.build_workload(a.config, 1, None)
    ex = FcpExecutor(result, 0, w.model, dev)
    _, (q, k, v, do) = bench.rank_inputs(ex, 0, w.model, dev)
    op = ex.op
    o, lse = ex.forward(q, k, v)
    prep = op.backward_prepare(o, lse, do)
    dk_b = torch.empty_like(k)
    dv_b = torch.empty_like(v)
    outs = op.alloc_forward_outputs()
    runs = {
        "fwd": lambda: op.forward_wave(0, q, k, v, None, None, outs),
        "bwd": lambda: op.backward_launch(False, q, k, v, None, None, prep, do, None, None, None, None,
                                          dk_out=dk_b, dv_out=dv_b),
        "dq": lambda: op.backward_dq(q, k, v, None, None, prep, do),
    }
    res = {}
    for name in a.kernels.split(","):
        fn = runs[name]
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        res[name] = sorted(ts)[len(ts) // 2]
    print(json.dumps({"config": a.config, "lib": os.environ.get("FCPB_LIB", "default"),
                      "ms": {k_: round(v_, 4) for k_, v_ in res.items()}}), flush=True)


if __name__ == "__main__":
    main()
