"""Probe: torch symmetric memory peer buffers + copy-engine pulls over NVLink (torchrun)."""
import os, time
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
try:
    symm.set_backend("CUDA")
except Exception as e:
    print("set_backend:", e)
n = 64 << 20   # 64 Mi bf16 = 128 MB
buf = symm.empty(n, dtype=torch.bfloat16, device=dev)
h = symm.rendezvous(buf, dist.group.WORLD)
buf.fill_(rank + 1)
h.barrier()
peer = (rank + 1) % world
src = h.get_buffer(peer, (n,), torch.bfloat16)
dst = torch.empty(n, dtype=torch.bfloat16, device=dev)
s = torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for k in range(64):   # 64 pulls of 2 MB (chunk-sized)
            a = k * (n // 64)
            dst[a:a + n // 64].copy_(src[a:a + n // 64], non_blocking=True)
    s.synchronize()
    dt = time.perf_counter() - t0
print(f"rank {rank}: pulled {n*2/1e6:.0f} MB from {peer} in {dt*1e3:.2f} ms = {n*2/dt/1e9:.0f} GB/s; ok={bool((dst == peer + 1).all())}", flush=True)
h.barrier()
dist.destroy_process_group()
