"""Summarise an ncu source page (`ncu -i X.ncu-rep --page source --csv --print-source sass`):
warp-stall samples per stall reason over the whole kernel, and the SASS instructions that
collect the most samples with their dominant reasons.

    python scripts/ncu_source_summary.py SOURCE.csv [--top 40] [--json OUT]
"""
import argparse
import csv
import json
from collections import Counter


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    body = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    si = hdr.index("Source")
    ni = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "(Not Issued)" not in h]
    tot = Counter()
    per = []
    for r in body:
        try:
            n = int(float(r[ni] or 0))
        except ValueError:
            continue
        st = Counter()
        for i in stall_cols:
            try:
                v = int(float(r[i] or 0))
            except ValueError:
                v = 0
            if v:
                st[hdr[i]] += v
                tot[hdr[i]] += v
        per.append((n, r[0], r[si].strip(), st))
    total = sum(n for n, *_ in per) or 1
    print(f"total samples {total}")
    for k, v in tot.most_common():
        print(f"  {k:28s} {v:9d}  {100 * v / total:5.1f}%")
    per.sort(key=lambda t: -t[0])
    print(f"\ntop {a.top} instructions:")
    for n, addr, src, st in per[:a.top]:
        top = ", ".join(f"{k[6:]}={v}" for k, v in st.most_common(3))
        print(f"  {100 * n / total:5.2f}%  {src[:60]:60s} {top}")
    if a.json:
        json.dump({"total_samples": total, "by_reason": dict(tot.most_common()),
                   "top": [{"pct": 100 * n / total, "sass": src, "reasons": dict(st.most_common(4))}
                           for n, _, src, st in per[:a.top]]}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()


def by_line(path, top=40):
    """Per-CUDA-line samples from `--print-source cuda,sass` (rows with a line number)."""
    rows = list(csv.reader(open(path)))
    out, fname, hdr = [], None, None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            n = int(float(r[4] or 0))
        except (ValueError, IndexError):
            continue
        st = Counter()
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "(Not Issued)" not in h and i < len(r):
                try:
                    v = int(float(r[i] or 0))
                except ValueError:
                    v = 0
                if v:
                    st[h[6:]] += v
        out.append((n, f"{fname}:{r[0]}", r[1].strip(), st))
    total = sum(x[0] for x in out) or 1
    out.sort(key=lambda t: -t[0])
    for n, loc, src, st in out[:top]:
        print(f"{100 * n / total:5.2f}%  {loc:28s} {src[:70]:70s} {dict(st.most_common(3))}")


def by_opcode(path, top=25):
    """Samples and executed warp instructions per SASS opcode (``--print-source sass``)."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    si, ni, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    samp, ex = Counter(), Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        samp[op] += int(float(r[ni] or 0))
        ex[op] += int(float(r[ei] or 0))
    tot_s, tot_e = sum(samp.values()) or 1, sum(ex.values()) or 1
    for op, n in samp.most_common(top):
        print(f"{op:14s} samples {100 * n / tot_s:5.1f}%   executed {ex[op]:12d} ({100 * ex[op] / tot_e:4.1f}%)")
