"""Benchmark / parity workloads C1-C5 (BASELINE.json ``configs``).

Each recipe returns the exact (lengths, tokens_per_worker, block, model) the
survey used to produce the reference's golden plan hashes, so the same batch is
rebuilt bit-for-bit on the GPU box without the reference package.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .costmodel import ModelConfig
from .workload import Batch, DistributionSpec, Sequence, generate_batch

TINY_MODEL = ModelConfig(q_heads=4, kv_heads=4, head_dim=64, dtype_bytes=4)
LLAMA3_8B = ModelConfig(q_heads=32, kv_heads=8, head_dim=128)


@dataclass(frozen=True)
class Workload:
    name: str
    lengths: tuple[int, ...]
    n_workers: int
    tokens_per_worker: int
    block_size: int
    model: ModelConfig

    def batch(self) -> Batch:
        return Batch(tuple(Sequence(i, n) for i, n in enumerate(self.lengths)),
                     self.n_workers, self.tokens_per_worker)

    @property
    def total_tokens(self) -> int:
        return sum(self.lengths)


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def c1_tiny(n: int = 2) -> Workload:
    lengths = tuple(int(x) for x in np.random.default_rng(0).integers(256, 4097, size=8))
    return Workload("C1-tiny", lengths, n, _ceil_div(sum(lengths), n), 512, TINY_MODEL)


def c2_llama8b_64k(n: int = 1) -> Workload:
    spec = DistributionSpec.lognormal(0.7, 4096, min_length=256, max_length=32768)
    lengths = tuple(s.length for s in generate_batch(spec, 0, 8, 8192).sequences)
    return Workload("C2-llama3-8b-64k", lengths, n, 65536 // n, 2048, LLAMA3_8B)


def c3_long_tail(n: int = 1) -> Workload:
    tail = np.random.default_rng(1).integers(1024, 8193, size=300)
    lengths = (262144,) + tuple(int(x) for x in tail)
    return Workload("C3-long-tail", lengths, n, _ceil_div(sum(lengths), n), 2048, LLAMA3_8B)


def c4_uniform_128k(n: int = 1) -> Workload:
    return Workload("C4-uniform-128k", (131072,) * n, n, 131072, 4096, LLAMA3_8B)


def c5_block_sweep(n: int = 1, block: int = 2048) -> Workload:
    spec = DistributionSpec.lognormal(0.7, 8192, min_length=512, max_length=32768)
    lengths = tuple(s.length for s in generate_batch(spec, 0, n, 32768).sequences)
    return Workload(f"C5-b{block}", lengths, n, 32768, block, LLAMA3_8B)


def by_name(name: str, n: int = 1, block: int | None = None) -> Workload:
    table = {"c1": c1_tiny, "c2": c2_llama8b_64k, "c3": c3_long_tail, "c4": c4_uniform_128k}
    key = name.lower()
    if key == "c5":
        return c5_block_sweep(n, block or 2048)
    return table[key](n)
