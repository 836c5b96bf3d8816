"""NVLink counters for the K5 copy-engine pulls, in ONE process on two GPUs so
ncu can profile it (ncu must never wrap a multi-rank command).

Rank 0's forward pull list of a real plan (`p2p.stage_pulls`, e.g. C3 at N=2) is replayed
with the product's own copy call (`native.copy_2d`, one 2-D copy-engine operation per merged
run) from a buffer on GPU 1 into a receive arena on GPU 0 -- the same bytes and copy shapes
the executor issues, with the peer region replaced by a same-process peer buffer.  The
copies sit inside a cudaProfilerStart/Stop range, so

    ncu --replay-mode range --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum \\
        python scripts/nvlink_ncu_probe.py --config c3 --world 2

reports the NVLink bytes of GPU 0 during the range; with ``--mode sm`` the same bytes move by
the K5 pull kernel (``fcpb_gather_copy``), which ncu also profiles in kernel mode.  Without
ncu it prints one JSON line with the CUDA-event GB/s of the same copies (plan bytes / time).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200 import native, p2p  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mode", default="ce", choices=["ce", "sm"],
                    help="ce: native.copy_2d per merged run; sm: the K5 pull kernel (fcpb_gather_copy)")
    ap.add_argument("--busy", action="store_true",
                    help="ce: time the pulls on a side stream while bf16 GEMMs keep every SM busy")
    a = ap.parse_args()
    assert torch.cuda.device_count() >= 2, "needs two GPUs in one process"
    w, result = bench.build_workload(a.config, a.world, None)
    Hk, D = w.model.kv_heads, w.model.head_dim
    row = Hk * D * 2
    pulls = [p for s in p2p.stage_pulls(result, a.rank) for p in s]
    src_rows = max(p.src + p.rows for p in pulls)
    dst_rows = max(p.dst + p.rows for p in pulls)
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    src = torch.randn((2, src_rows, Hk, D), device=d1).to(torch.bfloat16)
    dst = torch.zeros((2, dst_rows, Hk, D), device=d0, dtype=torch.bfloat16)
    torch.cuda.set_device(d0)
    if True:   # peer access 0 -> 1, as the IPC mapping gives the product path (kernel loads need
        # it; without it a copy-engine transfer between the GPUs is staged at ~30 GB/s)
        import ctypes
        import nvidia.cuda_runtime as crt
        rt = ctypes.CDLL(os.path.join(crt.__path__[0], "lib", "libcudart.so.12"))
        rt.cudaSetDevice(0)
        rc = rt.cudaDeviceEnablePeerAccess(1, 0)
        assert rc in (0, 704), f"cudaDeviceEnablePeerAccess: {rc}"   # 704: already enabled
    st = torch.cuda.current_stream(d0)
    nbytes = sum(p.rows for p in pulls) * 2 * row

    step = native.gather_seg_bytes()
    segs = [(dst.data_ptr() + pl * dst_rows * row + p.dst * row + o,
             src.data_ptr() + pl * src_rows * row + p.src * row + o, min(step, p.rows * row - o))
            for p in pulls for pl in range(2) for o in range(0, p.rows * row, step)]
    tab = torch.tensor(segs, dtype=torch.int64, device=d0)

    def pull_all():
        if a.mode == "sm":
            native.gather_copy(tab, 2 * 148, st)
            return
        for p in pulls:
            native.copy_2d(dst.data_ptr() + p.dst * row, dst_rows * row, src.data_ptr() + p.src * row,
                           src_rows * row, p.rows * row, 2, st)

    pull_all()                                   # warm
    torch.cuda.synchronize(d0)
    torch.cuda.synchronize(d1)
    for p in pulls[:8]:                          # spot-check the copied bytes
        assert torch.equal(dst[:, p.dst:p.dst + p.rows].cpu(), src[:, p.src:p.src + p.rows].cpu())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.busy:                                   # GEMMs on the default stream, pulls beside them
        side = torch.cuda.Stream(device=d0)
        x = torch.randn(8192, 8192, device=d0, dtype=torch.bfloat16)
        for _ in range(3):
            x @ x
        torch.cuda.synchronize(d0)
        for _ in range(20):                      # ~20 x 0.7 ms of tensor work queued first
            x @ x
        st = side
        torch.cuda.synchronize(d1)
    s.record(st)
    for _ in range(a.reps):
        pull_all()
    e.record(st)
    torch.cuda.synchronize(d0)
    ms = s.elapsed_time(e) / a.reps
    torch.cuda.synchronize(d0)
    torch.cuda.profiler.start()                  # the ncu range: one pass of the pull list
    pull_all()
    dst[0, 0, 0, :8].add_(0)                     # a kernel in the range (range replay needs one)
    torch.cuda.profiler.stop()
    torch.cuda.synchronize(d0)
    print(json.dumps({"what": "rank's forward pull list replayed GPU1 -> GPU0 with "
                              + ("native.copy_2d (copy engine)" if a.mode == "ce" else "the K5 pull kernel"),
                      "config": w.name, "world": a.world, "rank": a.rank, "copies": len(pulls),
                      "beside_busy_sms": a.busy,
                      "plan_bytes": nbytes, "mean_copy_MB": round(nbytes / len(pulls) / 1e6, 2),
                      "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9, "peak_GBps_per_direction": 900}),
          flush=True)


if __name__ == "__main__":
    main()
