"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel calls, total and per-call time."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[h.index("Kernel Name")][:70]
    agg[name][0] += 1
    agg[name][1] += float(r[h.index("Metric Value")].replace(",", ""))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0]:5d} {v[1] / 1000:10.1f} us total {v[1] / 1000 / v[0]:9.2f} us/call  {k}")
