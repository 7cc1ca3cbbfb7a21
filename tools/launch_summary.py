"""Summarise an ncu launch list (gpu__time_duration.sum CSV): time share per
kernel over the last `--tail` launches (e.g. the second of two solves).

    python tools/launch_summary.py launches.csv [--tail N]
"""
import argparse
import collections
import csv
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--tail", type=int, default=0)
ap.add_argument("--from-last", default=None,
                help="summarise from the last launch of this kernel (e.g. k_cheb_init)")
a = ap.parse_args()
rows = []
with open(a.csv) as f:
    lines = [l for l in f if l.startswith('"')]
for d in csv.DictReader(lines):
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("unnamed>::", "")
    rows.append((name, float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)))
if a.tail:
    rows = rows[-a.tail:]
if a.from_last:
    starts = [i for i, (n, _) in enumerate(rows) if n.startswith(a.from_last)]
    if starts:
        rows = rows[starts[-1]:]
agg = collections.defaultdict(lambda: [0, 0.0])
for n, us in rows:
    agg[n][0] += 1
    agg[n][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {tot / 1e3:.2f} ms serialized kernel time")
print(f"{'kernel':60s} {'n':>7s} {'total_ms':>9s} {'share':>6s} {'avg_us':>8s}")
for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n[:60]:60s} {c:7d} {us / 1e3:9.2f} {100 * us / tot:5.1f}% {us / c:8.2f}")
