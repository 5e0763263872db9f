"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python tools/launch_table.py LAUNCHES.csv [N]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
H = rows[h]
ki, vi = H.index("Kernel Name"), H.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    k = r[ki].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(r[vi])
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{k[:60]:60s} {n:5d} {t / 1e3:10.1f} us {t / tot * 100:5.1f}%")
print(f"total {tot / 1e3:.1f} us")
