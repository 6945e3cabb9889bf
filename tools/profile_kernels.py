"""Runs each SpMV kernel / transform of one BASELINE workload a few times, for
ncu captures (the numbers it prints are NOT bench values).

    python tools/profile_kernels.py --config 2 --reps 3 [--only crs,ell-inner]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--param", type=int, default=None)
ap.add_argument("--dparam", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", default="")
ap.add_argument("--transforms", action="store_true")
ap.add_argument("--formats", default="", help="comma list of formats to convert to")
ap.add_argument("--tune", default="", help="comma list of key=value tuning knobs")
a = ap.parse_args()
for kv in filter(None, a.tune.split(",")):
    k, v = kv.split("=")
    assert sp.load_library().spmvtk_k_tune(k.encode(), int(v)) == 0, kv
param = a.param or {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}[a.config]
only = set(a.only.split(",")) if a.only else None
sp.set_stream(torch.cuda.current_stream().cuda_stream)
m = sp.HostCrs(a.config, param, a.dparam).upload()
n = m.describe().n
fmts = {"coo-row": sp.Format.COO_ROW, "coo-col": sp.Format.COO_COL, "ell": sp.Format.ELL,
        "ell-row": sp.Format.ELL_ROWMAJOR, "ccs": sp.Format.CCS}
hs = {"crs": m}
fonly = set(a.formats.split(",")) if a.formats else None
for name, f in fmts.items():
    if fonly and name not in fonly:
        continue
    for _ in range(a.reps if a.transforms else 1):
        hs[name] = m.convert(f)
x = torch.ones(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ks = {"crs": ("crs", sp.Kernel.CRS), "coo-row": ("coo-row", sp.Kernel.COO_ROW_OUTER),
      "coo-col": ("coo-col", sp.Kernel.COO_COL_OUTER), "ell-inner": ("ell", sp.Kernel.ELL_INNER),
      "ell-outer": ("ell", sp.Kernel.ELL_OUTER), "ell-row": ("ell-row", sp.Kernel.ELL_ROWMAJOR)}
for name, (h, k) in ks.items():
    if (only and name not in only) or h not in hs:
        continue
    for _ in range(a.reps):
        hs[h].spmv_device(k, x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
print("done", n)
