"""A/B of the K3 LSE merge at C2 N=2's size (31,478 merged tokens x 32 heads, 1-4 partials
per group, mostly 2): one process per library variant (FCPB_LIB), CUDA-event time per
launch, and the max error against an fp64 torch merge of the same partials.

    FCPB_LIB=<variant .so> python scripts/micro/merge_ab.py
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2605_08524_b200 import native  # noqa: E402

H, D = 32, 128
lib = native.load(os.environ.get("FCPB_LIB"))
g = torch.Generator().manual_seed(3)
lens = [2098 + (i % 3) for i in range(15)]
nparts = [2, 2, 3, 2, 1, 2, 4, 2, 2, 3, 2, 2, 6, 2, 2]
groups, part_rows, rows, tok, q_off = [], [], 0, 0, 0
for L, n in zip(lens, nparts):
    groups.append([q_off, L, len(part_rows), len(part_rows) + n, tok, 0])
    for _ in range(n):
        part_rows.append(rows)
        rows += L
    tok += L
    q_off += L
M, P = tok, rows
op = torch.randn((P, H, D), generator=g).cuda()
lp = (torch.randn((P, H), generator=g) * 3).cuda()
lp[5, 3] = float("-inf")
gt = torch.tensor(groups, dtype=torch.int32).cuda()
pr = torch.tensor(part_rows, dtype=torch.int32).cuda()
o = torch.empty((M, H, D), dtype=torch.bfloat16, device="cuda")
lse = torch.empty((M, H), device="cuda")
a = native.MergeArgs()
a.num_q_heads, a.head_dim = H, D
a.o_partial, a.lse_partial = native.ptr(op), native.ptr(lp)
a.groups, a.num_groups = native.ptr(gt), len(groups)
a.part_rows, a.merged_tokens = native.ptr(pr), M
a.o, a.lse = native.ptr(o), native.ptr(lse)
st = torch.cuda.current_stream().cuda_stream


def run():
    native.check(lib.fcpb_lse_merge(ctypes.byref(a), st))


run()
torch.cuda.synchronize()
ref_o, ref_l = torch.empty((M, H, D), dtype=torch.float64), torch.empty((M, H), dtype=torch.float64)
opc, lpc = op.double().cpu(), lp.double().cpu()
for q0, L, pb, pe, _, _ in groups:
    ls = torch.stack([lpc[part_rows[s]:part_rows[s] + L] for s in range(pb, pe)])
    os_ = torch.stack([opc[part_rows[s]:part_rows[s] + L] for s in range(pb, pe)])
    lt = torch.logsumexp(ls, 0)
    ref_l[q0:q0 + L] = lt
    ref_o[q0:q0 + L] = (torch.exp(ls - lt)[..., None] * os_).sum(0)
err_o = (o.double().cpu() - ref_o).abs().max().item()
err_l = (lse.double().cpu() - ref_l).abs().max().item()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
n, tot = 50, 0.0
for _ in range(n):
    flush.zero_()                       # partials (1.1 GB) exceed L2 anyway; flush for safety
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
ms = tot / n
by = P * H * (D * 4 + 4) + M * H * (D * 2 + 4)
print(f"{os.path.basename(os.environ.get('FCPB_LIB') or 'default')}: {ms * 1e3:.1f} us  "
      f"{by / ms / 1e6:.0f} GB/s  max|dO|={err_o:.2e} max|dLSE|={err_l:.2e}")
