"""CRS->CCS / CRS->COO-col: the stable two-level partition (kernels_ccs.cu,
forced with the "ccs_stable" knob) against the rank-by-row bucketed pipeline -- arrays
compared bitwise between the two (and against the C oracle on the small
shapes, duplicates included), kernel time of each.

    python tools/tune_ccs.py [--configs 2,3,4,5] [--reps 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,4,5")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--dparams", default="0.0,1.0,2.0")
a = ap.parse_args()
lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}


def arrays(h, coo):
    out = [h.array(sp.Array.VALUES).view(np.uint64), h.array(sp.Array.ROW_IDX, 4, 0)]
    out.append(h.array(sp.Array.COL_IDX, 4, 0) if coo else h.array(sp.Array.POINTER, 4, 0))
    return out


def compare(m, label):
    for fmt, coo in ((sp.Format.CCS, False), (sp.Format.COO_COL, True)):
        lib.spmvtk_k_tune(b"ccs_stable", 1)
        new = m.convert(fmt)
        got = arrays(new, coo)
        lib.spmvtk_k_tune(b"ccs_stable", 0)
        old = m.convert(fmt)
        want = arrays(old, coo)
        same = all(np.array_equal(x, y) for x, y in zip(got, want))
        new.free()
        old.free()
        lib.spmvtk_k_tune(b"ccs_stable", 1)
        t_new = m.transform_kernel_seconds(fmt, a.reps)
        lib.spmvtk_k_tune(b"ccs_stable", 0)
        t_old = m.transform_kernel_seconds(fmt, a.reps)
        lib.spmvtk_k_tune(b"ccs_stable", 0)
        d = m.describe()
        by = 28 * d.nnz + 12 * d.n if not coo else 32 * d.nnz + 16 * d.n
        print(f"{label} {'coo-col' if coo else 'ccs    '}: stable {t_new * 1e6:8.1f} us "
              f"({by / t_new / 1e9:6.0f} GB/s)  rank-by-row {t_old * 1e6:8.1f} us  "
              f"identical={same}", flush=True)


for cfg in [int(c) for c in a.configs.split(",")]:
    for dp in ([float(x) for x in a.dparams.split(",")] if cfg == 5 else [0.0]):
        m = sp.HostCrs(cfg, PARAM[cfg], dp).upload()
        compare(m, f"cfg{cfg} D={dp}")
        m.free()
