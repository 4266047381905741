"""Per-kernel table (average us per launch, launch count) from an ncu --csv launch list
(--metrics gpu__time_duration.sum):  python tools/launch_table.py gpurun_out/x.csv"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
rows = list(csv.reader(line for line in open(sys.argv[1]) if not line.startswith("==")))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= max(ki, vi, ui) or not r[vi]:
        continue
    us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    k = r[ki].split("(")[0][:90]
    t, c = agg.get(k, (0.0, 0))
    agg[k] = (t + us, c + 1)
for k, (t, c) in agg.items():
    print(f"{t / c:10.1f} us x{c:<3d} {k}")
