"""Median per-kernel metrics from `ncu --metrics ... --csv` output (scripts/ab_cycles.sh)."""
import csv
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    while rows and "Kernel Name" not in rows[0]:
        rows = rows[1:]
    if not rows:
        print(f, "no rows")
        continue
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    acc = defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].split("::")[-1]
        try:
            acc[(name, r[mi])].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    out = defaultdict(dict)
    for (name, m), vals in acc.items():
        vals.sort()
        out[name][m.split(".")[0].replace("sm__", "").replace("gpu__", "")] = vals[len(vals) // 2]
    print(f, {k: {m: round(v, 1) for m, v in d.items()} for k, d in out.items()})
