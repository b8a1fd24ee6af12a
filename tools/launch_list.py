#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total time and share of GPU time.

    python tools/launch_list.py gpurun_out/launches.csv "<command line>" > profiles/rNN_launches.txt
"""
import csv
import re
import sys
from collections import defaultdict


def main(path, cmd=""):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", r["Kernel Name"])
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-6)
    total = sum(v[1] for v in agg.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none {cmd}")
    print("# (cold-cache, serialised replays: compare SHARES, not absolute times)")
    for name, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:74]:<76}launches={cnt:5d} total_ms={ms:10.3f} share={ms / total * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
