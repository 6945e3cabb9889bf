"""CRS->CCS / COO-col kernel time under tuning knobs of the default pipeline,
with the arrays of every variant compared bitwise against the first one.

    python tools/tune_ccs_knobs.py --knob ccs_subrows=0,1 [--knob ccs_coarse=8,9]
                                   [--configs 2,4] [--reps 10] [--coo]
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
a = ap.parse_args()
lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}
knobs = [(k.split("=")[0], [int(v) for v in k.split("=")[1].split(",")]) for k in a.knob]
combos = list(itertools.product(*[v for _, v in knobs]))


def setk(combo):
    for (name, _), v in zip(knobs, combo):
        lib.spmvtk_k_tune(name.encode(), v)


def arrays(h, coo):
    out = [h.array(sp.Array.VALUES).view(np.uint64), h.array(sp.Array.ROW_IDX, 4, 0)]
    out.append(h.array(sp.Array.COL_IDX, 4, 0) if coo else h.array(sp.Array.POINTER, 4, 0))
    return out


fmts = [(sp.Format.CCS, False)] + ([(sp.Format.COO_COL, True)] if a.coo else [])
for cfg in [int(c) for c in a.configs.split(",")]:
    for dp in ([float(x) for x in a.dparams.split(",")] if cfg == 5 else [0.0]):
        m = sp.HostCrs(cfg, PARAM[cfg], dp).upload()
        d = m.describe()
        for fmt, coo in fmts:
            ref = None
            line = f"cfg{cfg} D={dp} {'coo-col' if coo else 'ccs'}:"
            for combo in combos:
                setk(combo)
                h = m.convert(fmt)
                got = arrays(h, coo)
                h.free()
                if ref is None:
                    ref = got
                same = all(np.array_equal(x, y) for x, y in zip(got, ref))
                t = m.transform_kernel_seconds(fmt, a.reps)
                by = 28 * d.nnz + 12 * d.n if not coo else 32 * d.nnz + 16 * d.n
                tag = ",".join(f"{n}={v}" for (n, _), v in zip(knobs, combo))
                line += f"  [{tag}] {t * 1e6:8.1f} us ({by / t / 1e9:5.0f} GB/s){'' if same else ' DIFFERENT'}"
            print(line, flush=True)
        m.free()
setk(combos[0])
