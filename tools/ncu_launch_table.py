"""Per-launch table from an ncu --csv metrics capture (one row per kernel
launch: time and DRAM bytes):  python tools/ncu_launch_table.py FILE.csv"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
launches = OrderedDict()
for r in rows[1:]:
    d = launches.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
tot = 0.0
for i, d in launches.items():
    t = d.get("gpu__time_duration.sum", 0.0)
    tot += t
    print(f"{i:>3} {d['name'][:44]:44s} {t / 1e3:9.1f} us  read {d.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB"
          f"  write {d.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")
print(f"    total {tot / 1e3:.1f} us")
