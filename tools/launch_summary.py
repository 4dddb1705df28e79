"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("bri::", "").replace("void ", "")
    name = name.split("(")[0].split("<")[0]
    v = float(r[vi].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
unit = rows[hdr_i + 1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else "?"
grand = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total':>12s} {'share':>7s}  (unit {unit})")
for name, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{name:40s} {cnt[name]:8d} {v:12.1f} {100 * v / grand:6.1f}%")
print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {grand:12.1f}")
