"""Same-box yardstick (optional): flashinfer's CUTLASS sm100 FMHA (fmha_varlen,
forward only, library code) on the exact C2 batch at N=1, beside our K1 forward kernel.
FLOPs = 4*Hq*D * visible causal pairs (the reference accounting).

    python scripts/yardstick_flashinfer_fwd.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08524_b200 import configs  # noqa: E402
from paper_2605_08524_b200.costmodel import batch_token_pairs  # noqa: E402


def main():
    import flashinfer
    from flashinfer.prefill import fmha_varlen
    w = configs.by_name("c2", 1)
    L = list(w.lengths)
    T, H, Hk, D = sum(L), w.model.q_heads, w.model.kv_heads, w.model.head_dim
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1234)
    mk = lambda h: torch.randn((T, h, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q, k, v = mk(H), mk(Hk), mk(Hk)
    off = torch.tensor([0] + torch.tensor(L).cumsum(0).tolist(), dtype=torch.int32, device=dev)
    t0 = time.time()
    o = fmha_varlen(q, k, v, off, off, max_qo_len=max(L), causal=True)
    torch.cuda.synchronize()
    first = time.time() - t0
    for _ in range(3):
        fmha_varlen(q, k, v, off, off, max_qo_len=max(L), causal=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        fmha_varlen(q, k, v, off, off, max_qo_len=max(L), causal=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    flops = w.model.flops_per_token_pair * batch_token_pairs(L, "causal")
    print(json.dumps({"yardstick": "flashinfer %s fmha_varlen (CUTLASS sm100) causal fwd (library)" % flashinfer.__version__,
                      "workload": w.name, "fwd_ms": ms, "tflops": flops / (ms / 1e3) / 1e12,
                      "frac_of_1692": flops / (ms / 1e3) / 1692e12, "first_call_s": first}))


if __name__ == "__main__":
    main()
