"""Probe: capture one FcpExecutor step (fwd+bwd, exchange included) in a CUDA graph, replay,
compare with eager outputs and time both.  torchrun for N>1."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w, r = bench.build_workload(os.environ.get("CFG", "c2"), world, None)
    ex = FcpExecutor(r, rank, w.model, dev)
    _, (q, k, v, do) = bench.rank_inputs(ex, rank, w.model, dev)
    for _ in range(3):
        ref = ex.step(q, k, v, do)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            ex.step(q, k, v, do)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = ex.step(q, k, v, do)
    g.replay()
    torch.cuda.synchronize()
    diff = max((a.float() - b.float()).abs().max().item() for a, b in zip(out, ref))

    def timeit(fn, n=20):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    te = timeit(lambda: ex.step(q, k, v, do))
    tg = timeit(g.replay)
    print(json.dumps({"rank": rank, "world": world, "max_abs_diff_graph_vs_eager": diff,
                      "eager_ms": te, "graph_ms": tg}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
