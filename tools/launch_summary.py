"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
`bench.py --steps 2 --warmup 1`: per kernel launch count and mean duration,
and the share of each kernel in the device-resident step.

usage: python tools/launch_summary.py launches_C2.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    agg.setdefault(name, []).append(float(r[vi]) / 1e3)
print(f"{'kernel':60s} {'n':>4s} {'mean_us':>9s} {'min_us':>9s}")
for k, v in agg.items():
    print(f"{k[:60]:60s} {len(v):4d} {sum(v) / len(v):9.1f} {min(v):9.1f}")
