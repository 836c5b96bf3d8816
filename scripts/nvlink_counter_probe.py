"""Probe: do NVML's NVLink throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX,
field ids 138/139, KiB) move with a copy-engine peer copy on this box?  Two GPUs, one process.

    python scripts/nvlink_counter_probe.py
"""
import time

import pynvml
import torch

TX, RX = 138, 139


def field(h, fid, scope):
    v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
    if v.nvmlReturn != 0:
        return None
    return int(v.value.ullVal)


def main():
    pynvml.nvmlInit()
    h0 = pynvml.nvmlDeviceGetHandleByIndex(0)
    h1 = pynvml.nvmlDeviceGetHandleByIndex(1)
    nbytes = 4 << 30
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    torch.cuda.synchronize()
    scopes = list(range(18)) + [0xFFFFFFFF]
    before = {(d, f, s): field(h, f, s) for d, h in ((0, h0), (1, h1)) for f in (TX, RX) for s in scopes}
    t0 = time.perf_counter()
    for _ in range(4):
        b.copy_(a, non_blocking=True)          # GPU0 -> GPU1 over NVLink (copy engine)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    after = {(d, f, s): field(h, f, s) for d, h in ((0, h0), (1, h1)) for f in (TX, RX) for s in scopes}
    moved = 4 * nbytes
    print(f"copied {moved / 1e9:.1f} GB in {dt * 1e3:.1f} ms ({moved / dt / 1e9:.0f} GB/s wall)")
    for (d, f, s), v0 in before.items():
        v1 = after[(d, f, s)]
        if v0 is None or v1 is None:
            continue
        delta = v1 - v0
        if delta:
            print(f"gpu{d} {'TX' if f == TX else 'RX'} scope {s:#x}: +{delta} KiB = {delta * 1024 / 1e9:.2f} GB")
    ok = [k for k, v in before.items() if v is not None]
    print(f"{len(ok)} of {len(before)} (gpu, field, scope) reads succeeded")


if __name__ == "__main__":
    main()


def streams_probe():
    """Copy-engine peer pull bandwidth GPU1 <- GPU0 with the transfer split over k streams."""
    nbytes = 1 << 30
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    with torch.cuda.device(1):
        for k in (1, 2, 4, 8):
            streams = [torch.cuda.Stream(device=1) for _ in range(k)]
            part = nbytes // k
            for rep in range(3):
                torch.cuda.synchronize(1)
                t0 = time.perf_counter()
                for i, st in enumerate(streams):
                    with torch.cuda.stream(st):
                        dst[i * part:(i + 1) * part].copy_(src[i * part:(i + 1) * part], non_blocking=True)
                for st in streams:
                    st.synchronize()
                dt = time.perf_counter() - t0
            print(f"{k} stream(s): {nbytes / dt / 1e9:.0f} GB/s (1 GiB, last of 3)")


if __name__ == "__main__":
    streams_probe()
