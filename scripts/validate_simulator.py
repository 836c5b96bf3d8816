"""the reference's analytic simulate() (here simmodel, bit-identical) against
the measured B200 step times of profiles/r01_measured_configs.jsonl.  Predicted step =
simulate(fwd) + simulate(bwd: compute x2.5), with the reference's DEFAULT_EFFICIENCY and
with the B200-measured B200_EFFICIENCY, B200_HARDWARE (1692 TFLOP/s, 900 GB/s).

    python scripts/validate_simulator.py > profiles/r01_simulator_validation.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08524_b200.costmodel import B200_EFFICIENCY, B200_HARDWARE, DEFAULT_EFFICIENCY  # noqa: E402
from paper_2605_08524_b200.simmodel import SimOptions, simulate  # noqa: E402

NAMES = {"C2-llama3-8b-64k": "c2", "C3-long-tail": "c3", "C4-uniform-128k": "c4"}


def predict(r, cfg, curve):
    f = simulate(r.assignment, r.plan, r.units, r.deps, B200_HARDWARE, cfg, curve, SimOptions())
    b = simulate(r.assignment, r.plan, r.units, r.deps, B200_HARDWARE, cfg, curve, SimOptions(backward=True))
    return (f.total_time + b.total_time) * 1e3


def main():
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "profiles", "r01_measured_configs.jsonl")
    rows = []
    for line in open(src):
        if not line.strip():
            continue
        d = json.loads(line)
        wl, n, block = d["config"]["workload"], d["n_gpus"], d["config"]["block"]
        name = NAMES.get(wl, "c5")
        w, r = bench.build_workload(name, n, block if name == "c5" else None)
        pd, pb = predict(r, w.model, DEFAULT_EFFICIENCY), predict(r, w.model, B200_EFFICIENCY)
        rows.append({"workload": wl, "n": n, "block": block, "measured_ms": round(d["ms_per_step"], 3),
                     "sim_default_curve_ms": round(pd, 3), "sim_b200_curve_ms": round(pb, 3),
                     "ratio_default": round(d["ms_per_step"] / pd, 3),
                     "ratio_b200": round(d["ms_per_step"] / pb, 3)})
    print(json.dumps({"what": "measured / simulated step time (fwd+bwd)", "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
