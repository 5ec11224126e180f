#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel the
launch count, mean/total device time and share of the profiled process's GPU time.
(ncu launches are serialised and cold-cache: compare SHARES, not absolutes.)

usage: launches_summary.py launches.csv [--json out.json]
"""
import csv
import json
import sys
from collections import defaultdict


def summarise(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        rows.append((r["Kernel Name"], ns))
    agg = defaultdict(lambda: [0, 0.0])
    for name, ns in rows:
        short = name.split("(")[0].replace("void ", "")
        agg[short][0] += 1
        agg[short][1] += ns
    total = sum(v[1] for v in agg.values())
    out = []
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append({"kernel": k, "launches": n, "mean_us": ns / n / 1e3, "total_us": ns / 1e3,
                    "share": ns / total if total else 0.0})
    return out


def main():
    res = summarise(sys.argv[1])
    for r in res:
        print(f"{r['share'] * 100:6.2f}%  {r['launches']:5d} x {r['mean_us']:10.2f} us  {r['kernel']}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
