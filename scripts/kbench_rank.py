"""Per-kernel timing of ONE rank's work lists of an N-rank plan on one GPU (no exchange: the
receive arena holds random K/V), to study kernel efficiency as per-rank work shrinks.  Builds
the work lists exactly as FcpExecutor does at N>1 (one forward wave, fuse_remote="all").
Prints per-kernel ms, tile counts and the ideal time at the N=1 per-tile rate.  Under ncu add
sm__cycles_elapsed.max / smsp__cycles_active.avg for the launch tail.

    python scripts/kbench_rank.py [--config c2] [--world 4] [--rank 0] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.attention import BlockAttention  # noqa: E402
from paper_2605_08524_b200.worklist import build_rank_work  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--world", type=int, default=4)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--kernels", default="fwd,bwd,dq")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    w, result = bench.build_workload(a.config, a.world, None)
    fuse = "all" if a.world > 1 else False
    work = build_rank_work(result, a.rank, fuse_remote=fuse) if fuse else build_rank_work(result, a.rank)
    op = BlockAttention(work, w.model, dev)
    g = torch.Generator(device=dev).manual_seed(7)
    T, R = op.tokens, op.recv_tokens
    H, Hk, D = w.model.q_heads, w.model.kv_heads, w.model.head_dim
    rn = lambda *s: torch.randn(s, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q, k, v, do = rn(T, H, D), rn(T, Hk, D), rn(T, Hk, D), rn(T, H, D)
    kr, vr = (rn(R, Hk, D), rn(R, Hk, D)) if R else (None, None)
    outs = op.alloc_forward_outputs()

    def fwd():
        for i in range(op.num_waves):
            op.forward_wave(i, q, k, v, kr, vr, outs)
        op.merge(outs)

    fwd()
    prep = op.backward_prepare(outs[0], outs[1], do)
    f32 = lambda n: torch.zeros((max(n, 1), Hk, D), dtype=torch.float32, device=dev)
    dk, dv, dkr, dvr = f32(T), f32(T), f32(R), f32(R)
    dk_b, dv_b = torch.empty_like(k), torch.empty_like(v)

    def bwd():
        if R:
            op.backward_launch(True, q, k, v, kr, vr, prep, do, dk, dv, dkr, dvr)
        op.backward_launch(False, q, k, v, kr, vr, prep, do, dk, dv, dkr, dvr, dk_out=dk_b, dv_out=dv_b)

    runs = {"fwd": fwd, "bwd": bwd, "dq": lambda: op.backward_dq(q, k, v, kr, vr, prep, do)}
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
        res[name] = round(sorted(ts)[len(ts) // 2], 4)
    fw = work.fwd
    print(json.dumps({"config": a.config, "world": a.world, "rank": a.rank, "tokens": T, "recv_tokens": R,
                      "fwd_waves": len(fw.waves), "fwd_items": int(sum(len(x.items) for x in fw.waves)),
                      "ds_mode": op.ds_mode, "ms": res}), flush=True)


if __name__ == "__main__":
    main()
