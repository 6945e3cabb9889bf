"""Summarises an ncu --csv launch list (gpu__time_duration, dram bytes) per
kernel: count, mean time, DRAM bytes per launch, achieved DRAM GB/s.
With --by-grid, launches are keyed by (kernel, grid size), which separates
the same kernel on different matrices (configs)."""
import csv
import sys
from collections import OrderedDict

by_grid = "--by-grid" in sys.argv
rows = list(csv.reader(open([a for a in sys.argv[1:] if not a.startswith("--")][0])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
launch = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")
    if by_grid and "Grid Size" in ix:
        name = name[:38] + " " + r[ix["Grid Size"]].replace('"', "")
    key = (r[ix["ID"]], name[:48])
    d = launch.setdefault(key, {})
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    if unit == "Kbyte":
        v *= 1e3
    elif unit == "Mbyte":
        v *= 1e6
    elif unit == "Gbyte":
        v *= 1e9
    elif unit == "usecond":
        v *= 1e3
    elif unit == "msecond":
        v *= 1e6
    d[r[ix["Metric Name"]]] = v
agg = OrderedDict()
for (_, name), d in launch.items():
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
total = sum(a[1] for a in agg.values())
print(f"{'kernel':50s} {'n':>3s} {'mean us':>9s} {'share':>6s} {'DRAM MB':>9s} {'DRAM GB/s':>9s}")
for name, (c, t, b) in agg.items():
    print(f"{name:50s} {c:3d} {t / c / 1e3:9.1f} {t / total:6.1%} {b / c / 1e6:9.1f} "
          f"{(b / c) / (t / c) if t else 0:9.0f}")
