"""Per-phase timeline of the reshuffler's to-FCP move (C2, torchrun N ranks): local copies,
publish, the "published" barrier, the remote pulls and the final barrier, CUDA events on the
streams they run on (median of 5, each rank).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/reshuffle_probe.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.reshuffle import Reshuffler, user_layouts  # noqa: E402


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    w, r = bench.build_workload("c2", world, None)
    m = w.model
    rs = Reshuffler(r, rank, m, dev)
    T = rs.plan.user_tokens
    g = torch.Generator(device=dev).manual_seed(rank)
    mk = lambda h: torch.randn((T, h, m.head_dim), generator=g, device=dev).to(torch.bfloat16)
    usr = [mk(m.q_heads), mk(m.kv_heads), mk(m.kv_heads)]
    views = rs.input_views([(tuple(x.shape[1:]), x.dtype) for x in usr])
    for a, b in zip(views, usr):
        a.copy_(b)
    rows = []
    for it in range(6):
        dist.barrier()
        torch.cuda.synchronize()
        rs.marks = []
        rs.to_fcp(*views)
        torch.cuda.synchronize()
        t0 = rs.marks[0][1]
        if it:
            rows.append({n: round(t0.elapsed_time(e), 3) for n, e in rs.marks})
        rs.marks = None
    med = {k: sorted(x[k] for x in rows)[len(rows) // 2] for k in rows[0]}
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, "user_tokens": T, "fcp_tokens": rs.plan.fcp_tokens,
                                 "remote_bytes": rs.bytes_moved // 6, "phases_ms": med})
    if rank == 0:
        for o in out:
            print(json.dumps(o))
    rs.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
