"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python tools/launch_agg.py LAUNCHES.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
agg = collections.defaultdict(lambda: [0, 0.0])
order = []
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).split("::")[-1]
    v = float(r[h.index("Metric Value")].replace(",", "")) / 1e3
    agg[name][0] += 1
    agg[name][1] += v
    order.append((name, v))
tot = sum(t for n, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} n={n:6d} total_us={t:11.0f} avg_us={t / n:9.1f} share={t / tot:6.1%}")
