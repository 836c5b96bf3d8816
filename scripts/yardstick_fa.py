"""Same-box yardstick (optional): flash_attn 2.8 varlen causal fwd+bwd (FA2
algorithm, library kernels) on the exact C2 batch at N=1, with the same FLOP accounting as
bench.py (3.5 * 4*Hq*D * visible pairs).  Library code, reported beside our kernels only.

    python scripts/yardstick_fa.py [--config c2] [--steps 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08524_b200 import configs  # noqa: E402
from paper_2605_08524_b200.costmodel import batch_token_pairs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    from flash_attn import flash_attn_varlen_func
    w = configs.by_name(a.config, 1)
    L = list(w.lengths)
    T, H, Hk, D = sum(L), w.model.q_heads, w.model.kv_heads, w.model.head_dim
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1234)
    mk = lambda h: torch.randn((T, h, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q, k, v, do = mk(H), mk(Hk), mk(Hk), mk(H)
    q.requires_grad_(True); k.requires_grad_(True); v.requires_grad_(True)
    cu = torch.tensor([0] + list(torch.tensor(L).cumsum(0).tolist()), dtype=torch.int32, device=dev)
    mx = max(L)

    def step():
        o = flash_attn_varlen_func(q, k, v, cu, cu, mx, mx, causal=True)
        o.backward(do)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.steps
    flops = 3.5 * w.model.flops_per_token_pair * batch_token_pairs(L, "causal")
    print(json.dumps({"yardstick": "flash_attn %s varlen causal fwd+bwd (library)" % __import__("flash_attn").__version__,
                      "workload": w.name, "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
                      "tflops": flops / (ms / 1e3) / 1e12, "mfu_of_1692": flops / (ms / 1e3) / 1692e12}))


if __name__ == "__main__":
    main()
