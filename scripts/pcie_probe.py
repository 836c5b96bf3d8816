"""PCIe probe: H2D / D2H / both directions at once, with the copy split over 1, 2, 4 streams
(pinned host memory, 1.29 GB like one C2 step's inputs)."""
import time
import torch

N = 1289338880 // 2
dev = torch.device("cuda")
h = [torch.empty(N, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
d = [torch.empty(N, dtype=torch.bfloat16, device=dev) for _ in range(2)]


def run(k, mode):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, s in enumerate(streams):
        a, b = i * N // k, (i + 1) * N // k
        with torch.cuda.stream(s):
            if mode in ("h2d", "both"):
                d[0][a:b].copy_(h[0][a:b], non_blocking=True)
            if mode in ("d2h", "both"):
                h[1][a:b].copy_(d[1][a:b], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for mode in ("h2d", "d2h", "both"):
    for k in (1, 2, 4):
        run(k, mode)
        t = min(run(k, mode) for _ in range(3))
        print(f"{mode:5s} streams={k}  {t*1e3:7.2f} ms  {N*2/t/1e9:6.1f} GB/s per direction")
