"""Per-rank measured compute vs the plan's balance, for the reference efficiency curve and the
B200-calibrated one (torchrun, one rank per GPU):

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 scripts/rank_balance.py c3
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200 import configs  # noqa: E402
from paper_2605_08524_b200.api import ShardingConfig, fcp_schedule  # noqa: E402
from paper_2605_08524_b200.costmodel import B200_EFFICIENCY, DEFAULT_EFFICIENCY  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = configs.by_name(name, world, None)
    for label, curve in (("reference curve", DEFAULT_EFFICIENCY), ("b200 curve", B200_EFFICIENCY)):
        result = fcp_schedule(w.batch(), world, ShardingConfig(block_size=w.block_size), w.model, curve)
        ex = FcpExecutor(result, rank, w.model, dev)
        _, (q, k, v, do) = bench.rank_inputs(ex, rank, w.model, dev)
        rep = ex.measured_report(q, k, v, do, reps=2)
        if rank == 0:
            comp = [p.compute_time * 1e3 for p in rep.per_worker]
            print(f"{name} N={world} {label}: step {rep.total_time * 1e3:.1f} ms, per-rank compute ms "
                  + " ".join(f"{c:.1f}" for c in comp)
                  + f", max/mean {max(comp) / (sum(comp) / len(comp)):.3f}", flush=True)
        del ex
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
