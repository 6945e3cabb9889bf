"""Transform kernel time (CRS->CCS / COO-col by default; --formats for ELL,
ELL-row, COO-row) under tuning knobs, with the arrays of every variant
compared bitwise against the first one.

    python tools/tune_ccs_knobs.py --knob ccs_coarse=8,9 [--configs 2,4] [--reps 10] [--coo]
    python tools/tune_ccs_knobs.py --knob ell_wide_flat=0,1 --formats ell --configs 5
"""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,4,5")
ap.add_argument("--dparams", default="0.0,1.0,2.0")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--knob", action="append", default=[])
ap.add_argument("--coo", action="store_true")
ap.add_argument("--formats", default="", help="ell,ell-row,coo-row,ccs,coo-col (default ccs[,coo-col])")
a = ap.parse_args()
lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}
knobs = [(k.split("=")[0], [int(v) for v in k.split("=")[1].split(",")]) for k in a.knob]
combos = list(itertools.product(*[v for _, v in knobs]))


def setk(combo):
    for (name, _), v in zip(knobs, combo):
        lib.spmvtk_k_tune(name.encode(), v)


def arrays(h, kind):
    if kind == "ell":
        v, c = h.ell_bands(0, h.describe().band_count)
        return [v.view(np.uint64), c]
    if kind == "ell-row":
        return [h.array(sp.Array.VALUES).view(np.uint64), h.array(sp.Array.COL_IDX, 4, 0)]
    out = [h.array(sp.Array.VALUES).view(np.uint64), h.array(sp.Array.ROW_IDX, 4, 0)]
    out.append(h.array(sp.Array.COL_IDX, 4, 0) if kind != "ccs"
               else h.array(sp.Array.POINTER, 4, 0))
    return out


FMT = {"ccs": sp.Format.CCS, "coo-col": sp.Format.COO_COL, "coo-row": sp.Format.COO_ROW,
       "ell": sp.Format.ELL, "ell-row": sp.Format.ELL_ROWMAJOR}
names = a.formats.split(",") if a.formats else ["ccs"] + (["coo-col"] if a.coo else [])
fmts = [(FMT[k], k) for k in names]
for cfg in [int(c) for c in a.configs.split(",")]:
    for dp in ([float(x) for x in a.dparams.split(",")] if cfg == 5 else [0.0]):
        m = sp.HostCrs(cfg, PARAM[cfg], dp).upload()
        d = m.describe()
        for fmt, coo in fmts:
            ref = None
            line = f"cfg{cfg} D={dp} {coo}:"
            for combo in combos:
                setk(combo)
                h = m.convert(fmt)
                got = arrays(h, coo) if not (coo in ("ell", "ell-row") and d.nnz > (1 << 24)) else [np.zeros(1)]
                h.free()
                if ref is None:
                    ref = got
                same = all(np.array_equal(x, y) for x, y in zip(got, ref))
                t = m.transform_kernel_seconds(fmt, a.reps)
                by = {"ccs": 28 * d.nnz + 12 * d.n, "coo-col": 32 * d.nnz + 16 * d.n,
                      "coo-row": 28 * d.nnz + 4 * d.n}.get(coo, 12 * d.nnz + 4 * d.n)
                tag = ",".join(f"{n}={v}" for (n, _), v in zip(knobs, combo))
                line += f"  [{tag}] {t * 1e6:8.1f} us ({by / t / 1e9:5.0f} GB/s){'' if same else ' DIFFERENT'}"
            print(line, flush=True)
        m.free()
setk(combos[0])
