"""Same-box yardstick: the CuTe-DSL Blackwell flash
attention (FA4-style fwd/bwd for sm_100, shipped inside vllm as ``vllm_flash_attn.cute``;
library code) on the exact C2 batch at N=1 -- varlen causal, GQA 32/8, D=128, bf16 -- timed
separately for fwd and fwd+bwd, with bench.py's FLOP accounting (fwd 4*Hq*D per visible
pair, bwd 2.5x).  Reported beside our kernels only; never on the product path.

    python scripts/yardstick_fa4.py [--config c2] [--steps 20]
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
    from vllm.vllm_flash_attn.cute.interface import flash_attn_varlen_func
    w = configs.by_name(a.config, 1)
    L = list(w.lengths)
    T, H, Hk, D = sum(L), w.model.q_heads, w.model.kv_heads, w.model.head_dim
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1234)
    mk = lambda h: torch.randn((T, h, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q, k, v, do = mk(H), mk(Hk), mk(Hk), mk(H)
    q.requires_grad_(True)
    k.requires_grad_(True)
    v.requires_grad_(True)
    cu = torch.tensor([0] + list(torch.tensor(L).cumsum(0).tolist()), dtype=torch.int32, device=dev)
    mx = max(L)

    def fwd():
        out = flash_attn_varlen_func(q, k, v, cu_seqlens_q=cu, cu_seqlens_k=cu, max_seqlen_q=mx,
                                     max_seqlen_k=mx, causal=True)
        return out[0] if isinstance(out, tuple) else out

    def step():
        fwd().backward(do)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / a.steps

    ms_f = timed(lambda: fwd())
    ms = timed(step)
    ff = w.model.flops_per_token_pair * batch_token_pairs(L, "causal")
    print(json.dumps({"yardstick": "vllm_flash_attn.cute (CuTe-DSL sm100 FA4-style) varlen causal (library)",
                      "workload": w.name, "fwd_ms": ms_f, "fwd_tflops": ff / (ms_f / 1e3) / 1e12,
                      "ms_per_step": ms, "bwd_ms": ms - ms_f,
                      "bwd_tflops": 2.5 * ff / ((ms - ms_f) / 1e3) / 1e12,
                      "tokens_per_s": T / (ms / 1e3), "tflops": 3.5 * ff / (ms / 1e3) / 1e12}), flush=True)


if __name__ == "__main__":
    main()
