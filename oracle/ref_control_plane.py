"""TEST INFRASTRUCTURE ONLY: time the reference's own control plane (`fcp_schedule`, the
unmodified package pip-installed into ``baseline/_ref``) on one core, and emit its canonical
plan digest (SURVEY §8d "reference CPU path (i)"; Appendix A hash recipe, reference
``cli.py:214-250``).

Run as a separate interpreter whose import path holds only ``baseline/_ref`` (the repo's
``blocksched`` alias package would otherwise shadow the reference)::

    python oracle/ref_control_plane.py '{"lengths": [...], "n": 1, "tpw": 65536,
                                         "block": 2048, "model": {...}, "reps": 5}'

Prints one JSON object: ``{"ref_ms": median ms, "reps": k, "digest": sha256[:16]}``.
``run(...)`` launches it from ``bench.py`` and returns that dict (or ``{"unavailable": why}``).
"""
from __future__ import annotations

import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _child(spec: dict) -> dict:
    import blocksched as ref                      # baseline/_ref only (see run())
    from blocksched import cli
    assert os.path.dirname(os.path.dirname(ref.__file__)) == REF_DIR, ref.__file__
    model = ref.ModelConfig(**spec["model"])
    batch = ref.Batch(tuple(ref.Sequence(i, l) for i, l in enumerate(spec["lengths"])), spec["n"],
                      spec["tpw"])
    ts, r = [], None
    for _ in range(spec.get("reps", 5)):
        t0 = time.perf_counter()
        r = ref.fcp_schedule(batch, spec["n"], ref.ShardingConfig(block_size=spec["block"]), model,
                             ref.DEFAULT_EFFICIENCY)
        ts.append(time.perf_counter() - t0)
    blob = json.dumps([cli.schedule_payload(r, model), cli.plan_payload(r.sub_stage_plan, r.plan.degree)],
                      sort_keys=True)
    return {"ref_ms": statistics.median(ts) * 1e3, "reps": len(ts),
            "digest": hashlib.sha256(blob.encode()).hexdigest()[:16]}


def run(lengths, n, tpw, block, model_kw, reps=5, timeout=300) -> dict:
    if not os.path.isdir(os.path.join(REF_DIR, "blocksched")):
        return {"unavailable": "baseline/_ref not installed"}
    spec = json.dumps({"lengths": list(lengths), "n": n, "tpw": tpw, "block": block,
                       "model": model_kw, "reps": reps})
    env = dict(os.environ, PYTHONPATH=REF_DIR, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1",
               MKL_NUM_THREADS="1")
    # -I: isolated (no cwd / user site on sys.path); the reference is found via an explicit
    # sys.path entry only; taskset pins it to one core
    code = (f"import sys; sys.path.insert(0, {REF_DIR!r}); "
            f"sys.path.insert(1, {os.path.dirname(os.path.abspath(__file__))!r}); "
            "import ref_control_plane as m, json; print(json.dumps(m._child(json.loads(sys.argv[1]))))")
    cmd = [sys.executable, "-I", "-c", code, spec]
    try:
        cmd = ["taskset", "-c", str(sorted(os.sched_getaffinity(0))[0])] + cmd
    except Exception:
        pass
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=REF_DIR)
        if p.returncode != 0:
            return {"unavailable": (p.stderr.strip().splitlines() or ["failed"])[-1][:200]}
        out = json.loads(p.stdout.strip().splitlines()[-1])
        out["cores"] = 1
        return out
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


if __name__ == "__main__":
    print(json.dumps(_child(json.loads(sys.argv[1]))))
