"""TEST INFRASTRUCTURE ONLY: time the reference control plane (`fcp_schedule`, unmodified,
imported from /root/reference) next to this package's, on every SURVEY Appendix A recipe,
1 core each (SURVEY §8d "reference CPU path (i)").  Also checks the two plans are identical.
Writes profiles/r01_control_plane_timing.json.  Runs only where /root/reference exists.

    python -m oracle.time_control_plane
"""
from __future__ import annotations

import json
import os
import statistics
import time

from oracle import reference_plan
from paper_2605_08524_b200 import configs
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY
from paper_2605_08524_b200.pipeline import fcp_schedule, plan_digest
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.workload import Batch, Sequence


def _time(fn, reps):
    ts = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, out


def main():
    ref = reference_plan.load()
    rows = []
    cases = [("c1", 2, None)] + [(c, n, None) for c in ("c2", "c3") for n in (1, 2, 4, 8)] + \
            [("c4", n, None) for n in (1, 2, 4, 8)] + [("c5", 8, b) for b in (1024, 2048, 4096, 6144)]
    for name, n, block in cases:
        w = configs.by_name(name, n, block)
        batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(w.lengths)), n, w.tokens_per_worker)
        reps = 3 if name == "c3" else 7
        ours_ms, r = _time(lambda: fcp_schedule(batch, n, ShardingConfig(w.block_size), w.model,
                                                DEFAULT_EFFICIENCY), reps)
        model_kw = dict(q_heads=w.model.q_heads, kv_heads=w.model.kv_heads,
                        head_dim=w.model.head_dim, dtype_bytes=w.model.dtype_bytes)
        rb = ref.Batch(tuple(ref.Sequence(i, l) for i, l in enumerate(w.lengths)), n, w.tokens_per_worker)
        rm = ref.ModelConfig(**model_kw)
        ref_ms, _ = _time(lambda: ref.fcp_schedule(rb, n, ref.ShardingConfig(block_size=w.block_size), rm,
                                                    ref.DEFAULT_EFFICIENCY), reps)
        ref_hash, _ = reference_plan.reference_digest(list(w.lengths), n, w.tokens_per_worker,
                                                      w.block_size, model_kw)
        same = ref_hash == plan_digest(r, w.model)
        rows.append({"config": w.name, "n": n, "block": w.block_size, "ref_ms": round(ref_ms, 2),
                     "ours_ms": round(ours_ms, 2), "plans_identical": same})
        print(rows[-1], flush=True)
    out = {"what": "median wall time of fcp_schedule (host control plane), 1 core, this container",
           "cpu": os.uname().machine, "rows": rows}
    json.dump(out, open("profiles/r01_control_plane_timing.json", "w"), indent=1)


if __name__ == "__main__":
    main()
