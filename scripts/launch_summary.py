"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel.

usage: python scripts/launch_summary.py launches.csv "<command line>" > summary.txt
"""
import csv
import sys
from collections import defaultdict


def main(path, cmd):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1e3
        rows.append((r["Kernel Name"], us))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for k, us in rows:
        tot[k] += us
        cnt[k] += 1
    all_us = sum(tot.values())
    print(f"# {cmd}")
    print("# gpu__time_duration.sum per kernel (cold-cache, serialised by ncu), summed over the "
          "launches of warm-up + timed step")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k[:75]:75s} {cnt[k]:4d} launches {tot[k]:12.1f} us {100*tot[k]/all_us:6.1f}%  "
              f"({tot[k]/cnt[k]:10.2f} us/launch)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
