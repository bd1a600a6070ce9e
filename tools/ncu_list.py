"""Summarize an ncu --csv launch list: per-kernel durations in launch order."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
tot = 0.0
for r in rows[h + 1:]:
    v = float(r[vi].replace(",", "")) / 1e3; tot += v
    print(f"{r[ki].split('(')[0][:40]:42s} {v:8.2f} us")
print("total", round(tot, 1))
