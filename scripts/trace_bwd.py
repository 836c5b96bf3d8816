"""Debug: run the C2 backward with the FCPB_TRACE build and print CTA 0's per-tile timeline."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_08524_b200 import native
native._LIB_PATH = os.path.abspath("dbg/libfcpb_trace.so")
import bench
from paper_2605_08524_b200.executor import FcpExecutor
w, r = bench.build_workload("c2", 1, None)
ex = FcpExecutor(r, 0, w.model, torch.device("cuda"))
_, (q, k, v, do) = bench.rank_inputs(ex, 0, w.model, torch.device("cuda"))
for _ in range(3):
    ex.step(q, k, v, do)
torch.cuda.synchronize()
lib = native.load()
EV = ["QdIssue", "QdGot", "SdpIssue", "PdsGot", "AccIssue", "SdpGot", "Loaded", "PfreeGot", "PdsArrive", "DqGot", "DqDone"]
T = 256
buf = (ctypes.c_ulonglong * (len(EV) * T))()
lib.fcpb_debug_bwd_trace(buf, len(EV) * T)
a = np.frombuffer(buf, dtype=np.uint64).reshape(len(EV), T).astype(np.int64)
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, -1)
print("tile " + " ".join(f"{e:>9s}" for e in EV))
for j in range(0, 120):
    print(f"{j:4d} " + " ".join(f"{a[e, j]:9d}" for e in range(len(EV))))
d = np.diff(a[EV.index("AccIssue"), 20:120])
print("median AccIssue period (cycles):", np.median(d))
