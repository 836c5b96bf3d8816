"""A/B of the backward preprocess kernel (K3 bwd_preprocess) at C2's size: one process per
library variant (FCPB_LIB), CUDA-event time per launch over 200 launches with inputs far
larger than L2 between them, plus a checksum so variants can be compared bit for bit.

    FCPB_LIB=dbg/libfcpb_u8_t32.so python scripts/micro/prep_ab.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2605_08524_b200 import native  # noqa: E402

T, H, D = 62956, 32, 128
lib = native.load(os.environ.get("FCPB_LIB"))
g = torch.Generator(device="cuda").manual_seed(1)
o = torch.randn((T, H, D), device="cuda", generator=g).bfloat16()
do = torch.randn((T, H, D), device="cuda", generator=g).bfloat16()
lse = torch.randn((T, H), device="cuda", generator=g)
t_pad = (T + 3) // 4 * 4
lse2 = torch.empty((H, t_pad), device="cuda")
delta = torch.empty((H, t_pad), device="cuda")
st = torch.cuda.current_stream().cuda_stream


def run():
    native.check(lib.fcpb_bwd_preprocess(native.ptr(o), native.ptr(do), native.ptr(lse), native.ptr(lse2),
                                         native.ptr(delta), t_pad, None, T, H, D, st))


for _ in range(20):
    run()
torch.cuda.synchronize()
n = 200
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / n
by = 2 * T * H * D * 2 + T * H * 4 * 3
cs = (delta[:, :T].double().sum().item(), lse2[:, :T].double().sum().item())
print(f"{os.path.basename(os.environ.get('FCPB_LIB') or 'default')}: {ms * 1e3:.1f} us  "
      f"{by / ms / 1e6:.0f} GB/s  checksum={cs}")
