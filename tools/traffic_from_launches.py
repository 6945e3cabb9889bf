"""Extracts per-launch DRAM traffic (read + write bytes) of the SpMV kernels
from an ncu launch-list CSV into profiles/traffic_*.json (read by bench.py
for roofline.traffic)."""
import csv
import json
import sys
from collections import defaultdict

src, config, dst = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
per = defaultdict(lambda: defaultdict(float))
names = {}
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ix["Metric Unit"]], 1)
    per[r[ix["ID"]]][r[ix["Metric Name"]]] = v
    names[r[ix["ID"]]] = r[ix["Kernel Name"]]
pats = [("CrsRows", "crs"), ("k_spmv_crs_seg", "crs"), ("k_spmv_coo_row", "coo-row"), ("k_spmv_coo_col", "coo-col"),
        ("k_spmv_ell_cm<", "ell-inner"), ("EllRowMajorRows", "ell-row")]
out = defaultdict(list)
for i, k in names.items():
    for pat, lab in pats:
        if pat in k and "k_spmv" in k:
            out[lab].append(per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"])
try:
    res = json.load(open(dst))
except Exception:
    res = {}
res["source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                 "dram__bytes_write.sum --clock-control none; bytes per launch, mean")
res[config] = {k: sum(v) / len(v) for k, v in out.items()}
if "ell-inner" in res[config]:
    res[config].setdefault("ell-outer", res[config]["ell-inner"])
json.dump(res, open(dst, "w"), indent=1)
print(res[config])
