"""Print an ncu --csv launch list (gpu__time_duration.sum) in launch order: kernel, us."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows[hdr + 1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except (ValueError, IndexError):
        continue
    if flt and flt not in r[ki]:
        continue
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1.0)
    print(r[ki].split("(")[0][:60], round(v * scale, 2))
