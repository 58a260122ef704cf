"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows[hdr_i + 1:]:
    if len(r) <= max(ki, mi, vi) or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':72s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:72s} {n:8d} {t:10.1f} {t / n:9.2f} {100 * t / tot:5.1f}%")
print(f"{'total':72s} {sum(v[0] for v in agg.values()):8d} {tot:10.1f}")
