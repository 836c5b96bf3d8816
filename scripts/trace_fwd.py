"""Debug: C2 N=1 forward with the FCPB_TRACE build; CTA 0's per-tile timeline and medians of
the chain's hand-offs (clock64 cycles)."""
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
    ex.forward(q, k, v)
torch.cuda.synchronize()
lib = native.load()
EV = ["KGot", "S0Issue", "P0Got", "Pv0Issue", "P1Got", "Pv1Issue", "S0Got", "P0Arr", "S1Got", "P1Arr", "SLd0", "Max0", "Exp0"]
T = 256
buf = (ctypes.c_ulonglong * (len(EV) * T))()
lib.fcpb_debug_fwd_trace(buf, len(EV) * T)
c = np.frombuffer(buf, dtype=np.uint64).reshape(len(EV), T).astype(np.int64)
t0 = c[c > 0].min()
c = np.where(c > 0, c - t0, -1)
print("tile " + " ".join(f"{e:>8s}" for e in EV))
for j in range(int(os.environ.get("NPRINT", "40"))):
    print(f"{j:4d} " + " ".join(f"{c[e, j]:8d}" for e in range(len(EV))))
lo, hi = 5, 200
E = {e: c[i, lo:hi] for i, e in enumerate(EV)}
ok = np.all(c[:, lo:hi + 1] >= 0, axis=0)[: hi - lo]
def med(x):
    return float(np.median(x[ok]))
print("median period Pv1Issue:", float(np.median(np.diff(c[EV.index("Pv1Issue"), lo:hi]))))
print("softmax h0 S0Got->P0Arr:", med(E["P0Arr"] - E["S0Got"]), " h1 S1Got->P1Arr:", med(E["P1Arr"] - E["S1Got"]))
print("P0Arr->P0Got (MMA wakes):", med(E["P0Got"] - E["P0Arr"]), " P1Arr->P1Got:", med(E["P1Got"] - E["P1Arr"]))
print("P0Got->Pv0Issue:", med(E["Pv0Issue"] - E["P0Got"]), " P1Got->Pv1Issue:", med(E["Pv1Issue"] - E["P1Got"]))
# S0(j+1) issue is recorded at index j+1; its result arrives as S0Got[j+1]
s0i, s0g = c[EV.index("S0Issue"), lo + 1:hi + 1], c[EV.index("S0Got"), lo + 1:hi + 1]
print("S0Issue(j+1)->S0Got(j+1):", float(np.median(s0g - s0i)))
print("Pv0Issue(j)->S0Got(j+1):", float(np.median(s0g - c[EV.index("Pv0Issue"), lo:hi])))
print("Pv1Issue(j)->S1Got(j+1):", float(np.median(c[EV.index("S1Got"), lo + 1:hi + 1] - c[EV.index("Pv1Issue"), lo:hi])))
print("P0Arr(j)->S0Got(j+1) (tensor leg of head 0's chain):", float(np.median(s0g - c[EV.index("P0Arr"), lo:hi])))
print("head 0: S0Got->SLd0", med(E["SLd0"] - E["S0Got"]), " SLd0->Max0", med(E["Max0"] - E["SLd0"]),
      " Max0->Exp0", med(E["Exp0"] - E["Max0"]), " Exp0->P0Arr", med(E["P0Arr"] - E["Exp0"]))
