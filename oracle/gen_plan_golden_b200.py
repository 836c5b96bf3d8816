"""TEST INFRASTRUCTURE ONLY: regenerate ``tests/golden/plan_hashes_b200_curve.json``.

The unmodified reference planner (``oracle/reference_plan.py``) run with the B200-measured
efficiency curve (``costmodel.B200_EFFICIENCY``'s anchors, passed to the reference's own
``EfficiencyCurve``) over the SURVEY Appendix A recipes at N=1/2/4/8.  ``bench.py --curve
b200`` plans with that curve, so its plans are pinned to the reference the same way.

    python oracle/gen_plan_golden_b200.py
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.reference_plan import reference_digest  # noqa: E402
from paper_2605_08524_b200 import configs  # noqa: E402
from paper_2605_08524_b200.costmodel import B200_EFFICIENCY  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "plan_hashes_b200_curve.json")


def main():
    anchors = [list(a) for a in B200_EFFICIENCY.anchors]
    cases = []
    for n in (1, 2, 4, 8):
        recipes = [configs.c2_llama8b_64k(n), configs.c3_long_tail(n), configs.c4_uniform_128k(n)]
        recipes += [configs.c5_block_sweep(n, b) for b in (1024, 2048, 4096, 6144)]
        for w in recipes:
            m = w.model
            model = dict(q_heads=m.q_heads, kv_heads=m.kv_heads, head_dim=m.head_dim,
                         dtype_bytes=m.dtype_bytes)
            h, _ = reference_digest(w.lengths, w.n_workers, w.tokens_per_worker, w.block_size,
                                    model, curve_anchors=anchors)
            cases.append({"name": w.name, "n": n, "block": w.block_size, "sha": h})
    with open(OUT, "w") as fh:
        json.dump({"generator": "oracle/gen_plan_golden_b200.py",
                   "source": "/root/reference/pkg/src/blocksched (unmodified)",
                   "curve_anchors": anchors, "cases": cases}, fh, indent=1)
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
