"""measure the B200 attention efficiency the reference's EfficiencyCurve
models (costmodel.py:63-127): fwd+bwd MFU of the real kernels on uniform batches of one
sequence length at N=1, block 2048 (Llama-3-8B GQA).  Lengths below the block become
varlen packs (rated at their shortest member); longer ones become zigzag pairs, which
the model rates at the block size.  Prints the measured points and the fitted
monotone curve.

    python scripts/calibrate_efficiency.py > profiles/r01_efficiency_calibration.json
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.configs import LLAMA3_8B  # noqa: E402
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, batch_token_pairs  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402
from paper_2605_08524_b200.pipeline import fcp_schedule  # noqa: E402
from paper_2605_08524_b200.sharding import ShardingConfig  # noqa: E402
from paper_2605_08524_b200.workload import Batch, Sequence  # noqa: E402

PEAK = 1692e12
BLOCK = 2048


def measure(lengths, steps=10):
    dev = torch.device("cuda", 0)
    T = sum(lengths)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(lengths)), 1, T)
    r = fcp_schedule(batch, 1, ShardingConfig(BLOCK), LLAMA3_8B, DEFAULT_EFFICIENCY)
    ex = FcpExecutor(r, 0, LLAMA3_8B, dev)
    _, (q, k, v, do) = bench.rank_inputs(ex, 0, LLAMA3_8B, dev)
    for _ in range(3):
        ex.step(q, k, v, do)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        ex.step(q, k, v, do)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    flops = 3.5 * LLAMA3_8B.flops_per_token_pair * batch_token_pairs(lengths, "causal")
    return ms, flops / (ms * 1e-3) / PEAK


def main():
    points = []
    for L in (256, 512, 1024, 2048, 4096, 8192, 16384):
        n = max(65536 // L, 4)
        ms, mfu = measure([L] * n)
        points.append({"length": L, "sequences": n, "step_ms": ms, "mfu": mfu,
                       "unit_rating": "pack" if L < BLOCK else f"pair (rated at {BLOCK})"})
        print(json.dumps(points[-1]), file=sys.stderr, flush=True)
    # fitted curve: packs at their length; pairs at the block size, taking the mean MFU of
    # the >= block lengths (the model rates every pair at the block); made monotone.
    anchors = [(p["length"], p["mfu"]) for p in points if p["length"] < BLOCK]
    pair = sum(p["mfu"] for p in points if p["length"] >= BLOCK) / sum(1 for p in points if p["length"] >= BLOCK)
    anchors.append((BLOCK, pair))
    mono, best = [], 0.0
    for x, y in anchors:
        best = max(best, min(y, 1.0))
        mono.append((x, round(best, 4)))
    print(json.dumps({"what": "fwd+bwd MFU (of 1692 TFLOP/s) on uniform batches, N=1, block 2048, "
                              "Llama-3-8B GQA; B200 power-capped clocks",
                      "points": points, "b200_curve_anchors": mono}, indent=1))


if __name__ == "__main__":
    main()
