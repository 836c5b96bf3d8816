"""Timeline of FcpExecutor.forward_user (C2, torchrun N ranks), overlap=True and False: the
reshuffler's phases (local copies, barriers, pulls; reshuffle.py marks) and the executor's
forward phases (PRE_WAVE, exchange, waves), CUDA events relative to the call's start.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/forward_user_probe.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402
from paper_2605_08524_b200.reshuffle import Reshuffler  # noqa: E402


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    w, r = bench.build_workload("c2", world, None)
    m = w.model
    rs = Reshuffler(r, rank, m, dev)
    ex = FcpExecutor(r, rank, m, dev, resident=rs.resident_chunks())
    T = rs.plan.user_tokens
    g = torch.Generator(device=dev).manual_seed(rank)
    mk = lambda h: torch.randn((T, h, m.head_dim), generator=g, device=dev).to(torch.bfloat16)
    usr = [mk(m.q_heads), mk(m.kv_heads), mk(m.kv_heads)]
    views = rs.input_views([(tuple(x.shape[1:]), x.dtype) for x in usr])
    for a, b in zip(views, usr):
        a.copy_(b)
    res = {}
    # the bench's interleaving first: to-FCP alone, move-then-forward, overlapped (ms each)
    inter = []
    for it in range(4):
        row = {}
        for mode in ("to3", "seq", "ovl"):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if mode == "to3":
                rs.to_fcp(*views)
            elif mode == "seq":
                ex.forward(*rs.to_fcp(*views))
            else:
                ex.forward_user(rs, *views, overlap=True)
            b.record()
            torch.cuda.synchronize()
            row[mode] = round(a.elapsed_time(b), 3)
        inter.append(row)
    res["interleaved"] = inter
    for overlap in (True, False):
        for it in range(4):
            dist.barrier()
            torch.cuda.synchronize()
            start = torch.cuda.Event(enable_timing=True)
            start.record()
            rs.marks, ex._marks = [], []
            ex.forward_user(rs, *views, overlap=overlap)
            end = torch.cuda.Event(enable_timing=True)
            end.record()
            torch.cuda.synchronize()
            if it == 3:
                evs = [("rs:" + n, e) for n, e in rs.marks] + [("ex:" + n, e) for n, e in ex._marks]
                res[f"overlap={overlap}"] = dict(sorted(((n, round(start.elapsed_time(e), 3)) for n, e in evs),
                                                        key=lambda x: x[1]), total=round(start.elapsed_time(end), 3))
            rs.marks, ex._marks = None, None
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, **res})
    if rank == 0:
        for o in out:
            print(json.dumps(o))
    ex.close()
    rs.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
