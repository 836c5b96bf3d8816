"""Probe: can two processes that share ONE GPU rendezvous torch symmetric memory (gloo
process group) and pull from each other's buffers with copy-engine memcpys and exchange
stream-memory-op flags?  (The driver's GPU test box has one GPU.)

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29555 scripts/probe_samedev.py
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
dist.init_process_group("gloo")
mode = os.environ.get("PROBE_MODE", "symm")
n = 1 << 20
ok = False
try:
    if mode == "symm":
        import torch.distributed._symmetric_memory as symm
        buf = symm.empty(n, dtype=torch.float32, device=dev)
        h = symm.rendezvous(buf, dist.group.WORLD)
        buf.fill_(rank + 1)
        torch.cuda.synchronize()
        dist.barrier()
        peer = (rank + 1) % world
        src = h.get_buffer(peer, (n,), torch.float32)
        dst = torch.empty(n, device=dev)
        dst.copy_(src)
        torch.cuda.synchronize()
        ok = bool((dst == peer + 1).all())
        print(f"[symm] rank {rank}: pulled from {peer}: ok={ok}", flush=True)
    else:
        from paper_2605_08524_b200 import ipc
        reg = ipc.IpcRegion(n * 4, dev)
        views = reg.exchange(dist.group.WORLD)
        mine = reg.tensor(torch.float32, (n,))
        mine.fill_(rank + 1)
        torch.cuda.synchronize()
        dist.barrier()
        peer = (rank + 1) % world
        dst = torch.empty(n, device=dev)
        dst.copy_(views[peer].tensor(torch.float32, (n,)))
        torch.cuda.synchronize()
        ok = bool((dst == peer + 1).all())
        print(f"[ipc] rank {rank}: pulled from {peer}: ok={ok}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"[{mode}] rank {rank}: FAILED {type(e).__name__}: {e}", flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
