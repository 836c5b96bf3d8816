"""NVLink evidence for the K5/K6 exchange: the isolated copy-engine pulls of one
FCP step (forward K/V pulls, backward dK/dV returns), repeated R times under torchrun, with
the hardware NVLink data counters of this rank's GPU read by `nvidia-smi nvlink -gt d`
before and after (NVML's throughput fields are unavailable on this image, r01 notes).
Reports plan bytes, counter bytes (rx/tx summed over links) and GB/s per direction against
900 GB/s.  Rank 0 prints one JSON line.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P scripts/nvlink_exchange.py [--config c3] [--reps 20]
"""
import argparse
import json
import os
import re
import subprocess
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402


def nvlink_counters(gpu: int):
    """(rx_bytes, tx_bytes) summed over the GPU's links, or None if unavailable."""
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(gpu)], capture_output=True,
                             text=True, timeout=30).stdout
    except Exception:  # noqa: BLE001
        return None, ""
    rx = tx = 0
    found = False
    for line in out.splitlines():
        m = re.search(r"Link \d+: Data (Tx|Rx): (\d+) KiB", line)
        if m:
            found = True
            v = int(m.group(2)) * 1024
            if m.group(1) == "Rx":
                rx += v
            else:
                tx += v
    return ((rx, tx) if found else None), out[:400]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    w, result = bench.build_workload(a.config, world, None)
    ex = FcpExecutor(result, rank, w.model, dev)
    x = ex.xchg
    b = ex.exchange_bytes()
    Hk, D = w.model.kv_heads, w.model.head_dim
    staging = torch.empty((2, max(ex.ret_tokens, 1), Hk, D), dtype=torch.float32, device=dev)
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = int(vis.split(",")[local]) if vis else local
    res = {}
    for name in ("fwd_kv_pull", "bwd_dkv_return"):
        which = "kv" if name == "fwd_kv_pull" else "part"
        for it in range(2):                       # warm, then measured
            torch.cuda.synchronize()
            dist.barrier()
            c0, raw = nvlink_counters(phys)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = a.reps if it else 1
            cs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            with torch.cuda.stream(ex.comm):
                s.record(ex.comm)
                for i in range(n):
                    x.barrier(which, 0)
                    cs[i][0].record(ex.comm)
                    if which == "kv":
                        for st in range(len(ex.stages)):
                            x.pull_stage(st, ex.kv_recv)
                    else:
                        x.pull_returns(ex.returns, staging, ex.ret_rows)
                    cs[i][1].record(ex.comm)
                    x.barrier(which, 1)
                e.record(ex.comm)
            torch.cuda.synchronize()
            c1, _ = nvlink_counters(phys)
        ms = s.elapsed_time(e) / a.reps
        copy_ms = sum(b.elapsed_time(c) for b, c in cs) / len(cs)   # the pulls alone, no barriers
        nbytes = b["fwd_recv"] if which == "kv" else b["bwd_recv"]
        rec = {"plan_bytes_received": nbytes, "ms": ms, "GBps_received": nbytes / (ms * 1e-3) / 1e9 if ms else None,
               "copies": (sum(len(st) for st in x.stage_pulls) if which == "kv" else None),
               "copy_ms": copy_ms, "GBps_copies_only": nbytes / (copy_ms * 1e-3) / 1e9 if copy_ms else None}
        if c0 is not None and c1 is not None:
            rx, tx = (c1[0] - c0[0]) / a.reps, (c1[1] - c0[1]) / a.reps
            rec.update({"counter_rx_bytes": rx, "counter_tx_bytes": tx,
                        "counter_rx_GBps": rx / (ms * 1e-3) / 1e9 if ms else None,
                        "counter_tx_GBps": tx / (ms * 1e-3) / 1e9 if ms else None})
        else:
            rec["counter"] = "unavailable: " + raw.replace("\n", " | ")[:200]
        res[name] = rec
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        print(json.dumps({"what": "isolated exchange of one step, copy-engine pulls from IPC peer regions, "
                                  "NVLink data counters from nvidia-smi nvlink -gt d around R repetitions",
                          "config": w.name, "n_gpus": world, "reps": a.reps,
                          "peak_GBps_per_direction": 900, "per_rank": allr}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
