"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
agg = collections.OrderedDict()
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for r in rows[h + 1 + skip:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    k = r[ki].split("(")[0][-60:]
    a = agg.setdefault(k, [0, 0.0, r[gi] if gi is not None else ""])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
for k, (c, t, g) in agg.items():
    print(f"{c:6d} {t / 1e3:10.1f} us  {g:>14s}  {k}")
print(f"total {tot / 1e3:.1f} us")
