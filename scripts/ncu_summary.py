"""Summarise an `ncu --set full` raw CSV (ncu -i X.ncu-rep --page raw --csv) into
profiles/traffic.json (per-launch DRAM bytes of each attention kernel, read by bench.py for
roofline.traffic) and print the headline metrics of every kernel.

usage: python scripts/ncu_summary.py RAW.csv [--source NAME] [--out profiles/traffic.json]
"""
import argparse
import csv
import json

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "cycles": ("sm__cycles_elapsed.max", 1),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", 1e-9),
    "tensor_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
    "mufu_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "registers": ("launch__registers_per_thread", 1),
    "smem_bytes": ("launch__shared_mem_per_block_dynamic", 1),
}
UNIT = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "Ghz": 1e9, "Mhz": 1e6, "hz": 1, "cycle": 1, "%": 1, "": 1, "register/thread": 1,
        "Kbyte/block": 1e3, "byte/block": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--source", default=None)
    ap.add_argument("--out", default="profiles/traffic.json")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
        rec = {}
        for k, (m, scale) in KEYS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1)
            except ValueError:
                continue
            if k == "duration_ms":
                v = v * 1e3
            elif k == "sm_ghz":
                v = v * 1e-9
            rec[k] = round(v, 4) if isinstance(v, float) else v
        if "dram_read_bytes" in rec:
            rec["traffic_bytes"] = rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0)
        out.setdefault(name, rec)              # first launch of each kernel
        print(name, rec)
    json.dump({"source": a.source or a.raw, "kernels": out}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
