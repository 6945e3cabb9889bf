"""SpMV kernel variants on BASELINE workloads (device time, CUDA events,
inputs larger than L2), each checked against the sub-warp CRS kernel.

    python tools/tune_spmv.py --configs 2,3,4,5 [--reps 50]

Prints one line per (config, kernel, variant); the numbers are tuning data,
not bench values.
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
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--dparam", type=float, default=0.0)
ap.add_argument("--crs", default="16,18,20")
ap.add_argument("--seg-ks", default="4", help="(only 4 remains: 8 entries per lane was slower)")
ap.add_argument("--seg-chunks", default="1024,2048,4096")
ap.add_argument("--coo", default="1,2")
ap.add_argument("--coo-chunks", default="1024,2048,4096")
ap.add_argument("--coo-segs", default="0")
ap.add_argument("--ell", type=int, default=1, help="also time ELL-inner (where it fits)")
a = ap.parse_args()
lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}


def tune(key, v):
    assert lib.spmvtk_k_tune(key.encode(), int(v)) == 0


def timed(h, k, x, y, reps):
    for _ in range(3):
        h.spmv_device(k, x.data_ptr(), y.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        h.spmv_device(k, x.data_ptr(), y.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


for cfg in [int(c) for c in a.configs.split(",")]:
    m = sp.HostCrs(cfg, PARAM[cfg], a.dparam).upload()
    d = m.describe()
    st = m.row_stats()
    n, nnz = d.n, d.nnz
    print(f"config {cfg} n={n} nnz={nnz} mean={nnz / n:.1f} max_row={st.max_row} "
          f"d_mat={st.d_mat:.4f}", flush=True)
    x = torch.from_numpy(sp.gen_vector(n, 7)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    tune("crs_variant", 16)
    m.spmv_device(sp.Kernel.CRS, x.data_ptr(), y.data_ptr())
    ref = y.cpu().numpy().copy()
    crs_bytes = 12 * nnz + 4 * (n + 1) + 16 * n
    for v in [int(s) for s in a.crs.split(",")]:
        tune("crs_variant", v)
        chunks = [int(c) for c in a.seg_chunks.split(",")] if v == 20 else [0]
        ks = [int(c) for c in a.seg_ks.split(",")] if v == 20 else [4]
        for dep, c in [(dd, cc) for dd in ks for cc in chunks]:
            tune("seg_chunk", c)
            y.fill_(np.nan)
            t = timed(m, sp.Kernel.CRS, x, y, a.reps)
            got = y.cpu().numpy()
            err = float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))
            print(f"    crs v{v:2d} k{dep} chunk={c:5d}: {t * 1e6:8.1f} us {crs_bytes / t / 1e9:7.0f} GB/s "
                  f"{nnz / t / 1e9:6.1f} Ggather/s err={err:.1e}", flush=True)
    tune("crs_variant", -1)
    tune("seg_chunk", 0)
    coo = m.convert(sp.Format.COO_ROW)
    coo_bytes = 16 * nnz + 16 * n
    for v in [int(s) for s in a.coo.split(",")]:
        tune("coo_variant", v)
        chunks = [int(c) for c in a.coo_chunks.split(",")] if v == 2 else [0]
        for sv, c in [(0, x2) for x2 in chunks]:
            tune("coo_chunk", c)
            y.fill_(np.nan)
            t = timed(coo, sp.Kernel.COO_ROW_OUTER, x, y, a.reps)
            got = y.cpu().numpy()
            err = float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))
            print(f"    coo v{v} s{sv} chunk={c:5d}: {t * 1e6:8.1f} us {coo_bytes / t / 1e9:7.0f} GB/s "
                  f"{nnz / t / 1e9:6.1f} Ggather/s err={err:.1e}", flush=True)
    tune("coo_variant", 1)
    tune("coo_chunk", 0)
    coo.free()
    if a.ell and st.max_row * n * 12 < (40 << 30):
        ell = m.convert(sp.Format.ELL)
        nz = ell.describe().band_count
        ell_bytes = 12 * n * nz + 16 * n
        y.fill_(np.nan)
        t = timed(ell, sp.Kernel.ELL_INNER, x, y, a.reps)
        got = y.cpu().numpy()
        err = float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))
        print(f"    ell inner : {t * 1e6:8.1f} us {ell_bytes / t / 1e9:7.0f} GB/s "
              f"{nnz / t / 1e9:6.1f} Ggather/s err={err:.1e}", flush=True)
        ell.free()
    m.free()
