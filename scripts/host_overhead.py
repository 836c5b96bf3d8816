"""Host enqueue time of one executor step (no synchronisation inside the timed call) vs the
device step time, per rank: shows whether the Python host side could starve the GPU.
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/host_overhead.py
"""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402


def main():
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w, r = bench.build_workload(os.environ.get("CFG", "c2"), world, None)
    ex = FcpExecutor(r, rank, w.model, dev)
    _, (q, k, v, do) = bench.rank_inputs(ex, rank, w.model, dev)
    for _ in range(3):
        ex.step(q, k, v, do)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    host = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        t0 = time.perf_counter()
        ex.step(q, k, v, do)
        host.append((time.perf_counter() - t0) * 1e3)
    e.record()
    torch.cuda.synchronize()
    out = {"rank": rank, "world": world, "host_enqueue_ms_median": sorted(host)[10],
           "host_enqueue_ms_max": max(host), "device_ms_per_step": s.elapsed_time(e) / 20,
           "launches_per_step": ex.op.launches / 23 if hasattr(ex.op, "launches") else None}
    print(json.dumps(out), flush=True)
    ex.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
