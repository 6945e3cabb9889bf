"""Summarise an ncu --csv metrics log: one line per launch, metrics side by side.

    python tools/ncu_csv_summary.py gpurun_out/x.csv
"""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = [l for l in open(path) if l.startswith('"')]
    r = list(csv.reader(rows))
    h = r[0]
    launches = OrderedDict()
    for row in r[1:]:
        d = dict(zip(h, row))
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("<unnamed>::", ""))
        launches.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
    for (i, name), m in launches.items():
        vals = "  ".join(f"{k.split('.')[0].split('__')[-1]}={v}" for k, v in m.items())
        print(f"{i:>3} {name[:36]:36s} {vals}")


if __name__ == "__main__":
    main(sys.argv[1])
