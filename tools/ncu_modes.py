"""Summarise an ncu launch list of tools/upd3_ablate.py: median duration (us) of the
matching kernel per (layer, mode) group of `reps` launches, in launch order (each
layer: one plan-resolving launch, then `modes` groups)."""
import csv
import sys

path, flt, reps, modes = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
v = []
for r in rows[hdr + 1:]:
    if flt not in r[ki]:
        continue
    x = float(r[vi].replace(",", ""))
    v.append(x / 1e3 if r[ui].startswith("n") else x)
per = 1 + modes * reps
for l0 in range(0, len(v), per):
    lay = v[l0 + 1:l0 + per]
    groups = [sorted(lay[i:i + reps]) for i in range(0, len(lay), reps)]
    print(" ".join("%.1f" % g[len(g) // 2] for g in groups))
