"""TEST INFRASTRUCTURE ONLY: regenerate ``tests/golden/plan_hashes.json``.

Runs the unmodified reference planner (``oracle/reference_plan.py``) over
(1) the SURVEY Appendix A recipes C1-C5 at every N and (2) a seeded random
corpus (lengths 1..20K, N 1..8, blocks 512..6144, both masks, several coalesce
degrees) and records the canonical plan hash of each case.  The product
planner is then checked against these hashes on any machine.

    python oracle/gen_plan_golden.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.reference_plan import reference_digest  # noqa: E402
from paper_2605_08524_b200 import configs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "plan_hashes.json")


def _model_kw(m):
    return dict(q_heads=m.q_heads, kv_heads=m.kv_heads, head_dim=m.head_dim,
                dtype_bytes=m.dtype_bytes)


def main(n_random: int = 1200):
    cases = []
    recipes = [configs.c1_tiny(2)]
    for n in (1, 2, 4, 8):
        recipes += [configs.c2_llama8b_64k(n), configs.c3_long_tail(n), configs.c4_uniform_128k(n)]
        recipes += [configs.c5_block_sweep(n, b) for b in (1024, 2048, 4096, 6144)]
    for w in recipes:
        h, _ = reference_digest(w.lengths, w.n_workers, w.tokens_per_worker, w.block_size,
                                _model_kw(w.model))
        cases.append({"name": w.name, "lengths": list(w.lengths), "n": w.n_workers,
                      "tpw": w.tokens_per_worker, "block": w.block_size,
                      "model": _model_kw(w.model), "mask": "causal", "coalesce": 16,
                      "sha": h})
    rng = np.random.default_rng(20261018)
    for k in range(n_random):
        n = int(rng.integers(1, 9))
        block = int(rng.choice([512, 1024, 2048, 4096, 6144]))
        count = int(rng.integers(1, 16))
        hi = int(rng.choice([2000, 8000, 20000]))
        lengths = [int(x) for x in rng.integers(1, hi + 1, size=count)]
        mask = "causal" if rng.random() < 0.85 else "full"
        coal = int(rng.choice([1, 4, 16]))
        tot = sum(lengths)
        tpw = -(-tot // n) if rng.random() < 0.7 else 1 << 20
        model = {"q_heads": 32, "kv_heads": 8, "head_dim": 128, "dtype_bytes": 2}
        try:
            h, _ = reference_digest(lengths, n, tpw, block, model, mask, coal)
        except Exception as exc:  # the reference raises: record the exception type
            h = "raise:" + type(exc).__name__
        cases.append({"name": f"rand{k}", "lengths": lengths, "n": n, "tpw": tpw,
                      "block": block, "model": model, "mask": mask, "coalesce": coal,
                      "sha": h})
    with open(OUT, "w") as fh:
        json.dump({"generator": "oracle/gen_plan_golden.py",
                   "source": "/root/reference/pkg/src/blocksched (unmodified)",
                   "cases": cases}, fh, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
