"""Print the headline fields of bench.py JSON lines (one per file): tokens/s, ms/step, MFU,
per-kernel ms and the SM clock.   python scripts/bench_summary.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([x for x in open(f) if x.startswith("{")][-1])
    except (IndexError, ValueError, OSError) as e:
        print(f, "no line", e)
        continue
    ks = {k.replace("attn_", "").replace("_kernel", ""): round(v["ms"], 3) for k, v in d.get("kernels", {}).items()}
    print(f"{f}: {d['value'] / 1e6:.3f}M tok/s {d['ms_per_step']:.2f} ms mfu {d.get('mfu', 0):.3f} {ks} "
          f"sm {d['clocks'].get('sm_mhz')} MHz")
