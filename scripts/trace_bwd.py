"""Debug: run the C2 backward with the FCPB_TRACE build and print CTA 0's per-tile timeline."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_08524_b200 import native
native._LIB_PATH = os.path.abspath(os.environ.get("FCPB_LIB", "dbg/libfcpb_trace.so"))
import bench
from paper_2605_08524_b200.executor import FcpExecutor
w, r = bench.build_workload("c2", 1, None)
ex = FcpExecutor(r, 0, w.model, torch.device("cuda"))
_, (q, k, v, do) = bench.rank_inputs(ex, 0, w.model, torch.device("cuda"))
for _ in range(3):
    ex.step(q, k, v, do)
torch.cuda.synchronize()
lib = native.load()
EV = ["QIssue", "QGot", "SIssue", "PGot", "DvIssue", "DsGot", "DkIssue", "SGot", "PArrive", "DpGot", "DsArrive", "SLd", "PSt", "DpLd", "DsSt"]
T = 256
buf = (ctypes.c_ulonglong * (len(EV) * T))()
lib.fcpb_debug_bwd_trace(buf, len(EV) * T)
a = np.frombuffer(buf, dtype=np.uint64).reshape(len(EV), T).astype(np.int64)
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, -1)
print("tile " + " ".join(f"{e:>9s}" for e in EV))
for j in range(0, int(os.environ.get("NPRINT", "120"))):
    print(f"{j:4d} " + " ".join(f"{a[e, j]:9d}" for e in range(len(EV))))
d = np.diff(a[EV.index("DkIssue"), 20:120])
print("median DkIssue period (cycles):", np.median(d))
for x, y in [("SGot", "PArrive"), ("DpGot", "DsArrive"), ("SIssue", "SGot"), ("SGot", "SLd"), ("SLd", "PSt"), ("PSt", "PArrive"), ("PArrive", "DpGot"), ("DpGot", "DpLd"), ("DpLd", "DsSt"), ("DsSt", "DsArrive"), ("DsArrive", "SGot"), ("PGot", "DvIssue"), ("DsGot", "DkIssue"), ("PArrive", "PGot"), ("DsArrive", "DsGot")]:
    print(f"median {x}->{y}:", np.median(a[EV.index(y), 20:120] - a[EV.index(x), 20:120]))
import time
s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(5):
    ex.step(q, k, v, do)
e0.record(); torch.cuda.synchronize()
print("step ms:", s0.elapsed_time(e0) / 5)

EV2 = ["KIssue", "KGot", "SIssue", "DsGot", "DqIssue", "SGot", "Freed", "DpGot", "DsArrive"]
buf2 = (ctypes.c_ulonglong * (len(EV2) * T))()
lib.fcpb_debug_dq_trace(buf2, len(EV2) * T)
b = np.frombuffer(buf2, dtype=np.uint64).reshape(len(EV2), T).astype(np.int64)
if not (b > 0).any():
    b[:] = 1      # materialised-dS mode: the recompute dQ kernel did not run
t0 = b[b > 0].min()
b = np.where(b > 0, b - t0, -1)
print("dq tile " + " ".join(f"{e:>9s}" for e in EV2))
for j in range(0, int(os.environ.get("NPRINT2", "30"))):
    print(f"{j:4d} " + " ".join(f"{b[e, j]:9d}" for e in range(len(EV2))))
d2 = np.diff(b[EV2.index("DqIssue"), 10:100])
print("dq median DqIssue period (cycles):", np.median(d2))

EV3 = ["KGot", "S0Issue", "P0Got", "Pv0Issue", "P1Got", "Pv1Issue", "S0Got", "P0Arr", "S1Got", "P1Arr"]
buf3 = (ctypes.c_ulonglong * (len(EV3) * T))()
lib.fcpb_debug_fwd_trace(buf3, len(EV3) * T)
c3 = np.frombuffer(buf3, dtype=np.uint64).reshape(len(EV3), T).astype(np.int64)
t0 = c3[c3 > 0].min()
c3 = np.where(c3 > 0, c3 - t0, -1)
print("fwd tile " + " ".join(f"{e:>8s}" for e in EV3))
for j in range(0, int(os.environ.get("NPRINT3", "20"))):
    print(f"{j:4d} " + " ".join(f"{c3[e, j]:8d}" for e in range(len(EV3))))
d3 = np.diff(c3[EV3.index("Pv1Issue"), 5:60])
print("fwd median period (cycles):", np.median(d3))
print("median DsArrive(j)->SGot(j+1):", np.median(a[EV.index("SGot"), 21:121] - a[EV.index("DsArrive"), 20:120]))
print("median DkIssue(j)->DpGot(j+1):", np.median(a[EV.index("DpGot"), 21:121] - a[EV.index("DkIssue"), 20:120]))
print("median DvIssue(j)->SGot(j+1):", np.median(a[EV.index("SGot"), 21:121] - a[EV.index("DvIssue"), 20:120]))
