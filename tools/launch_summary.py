"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file):
per-launch times of the LAST matvec and per-kernel shares.
    python tools/launch_summary.py launches.csv [title]"""
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
title = sys.argv[2] if len(sys.argv) > 2 else ""


def us(r):
    v = float(r["Metric Value"].replace(",", ""))
    u = r.get("Metric Unit", "")
    return v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v


# the last matvec: launches after the last k_set_density
starts = [i for i, r in enumerate(rows) if "k_set_density" in r["Kernel Name"]]
last = rows[starts[-1]:] if starts else rows
tot = sum(us(r) for r in last)
print(f"# ncu launch list, one matvec {title}, gpu__time_duration.sum, --clock-control none")
print("# cold-cache serialised per-launch times: compare shares, not absolutes")
print(f"# total {tot:.1f} us over {len(last)} launches")
for r in last:
    print(f"{us(r):10.1f} us {100 * us(r) / tot:6.1f}%  {r['Kernel Name'].split('(')[0]}")
agg = {}
for r in last:
    k = r["Kernel Name"].split("(")[0]
    agg[k] = agg.get(k, 0) + us(r)
print("# by kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / tot:6.1f}%  {k}")
