"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except (ValueError, IndexError):
        continue
    name = r[ki].split("(")[0] if "<" not in r[ki] else r[ki].split(">(")[0] + ">"
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
print("kernel,launches,total_ns,share")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k},{n},{int(v)},{v / tot:.4f}")
