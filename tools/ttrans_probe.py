"""Breaks down t_trans of CRS->ELL: the library's own measure_transformation
timing (spmvtk_matrix_convert_timed: device synchronised, wall clock around
the conversion) against the kernels alone, per config.

    SPMVTK_TRACE_ELL=1 python tools/ttrans_probe.py --configs 1,2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2")
ap.add_argument("--reps", type=int, default=15)
a = ap.parse_args()
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}
sp.set_stream(torch.cuda.current_stream().cuda_stream)
sp.reserve_device_memory(8 << 30)
for cfg in [int(c) for c in a.configs.split(",")]:
    m = sp.HostCrs(cfg, PARAM[cfg]).upload()
    for fmt in (sp.Format.ELL, sp.Format.ELL_ROWMAJOR, sp.Format.COO_ROW):
        for _ in range(3):
            m.convert(fmt).free()
        ts = []
        for _ in range(a.reps):
            h, t = m.convert_timed(fmt)
            ts.append(t)
            h.free()
        ts.sort()
        k = m.transform_kernel_seconds(fmt, a.reps)
        print(f"config {cfg} {fmt.name:13s}: t_trans median {ts[len(ts) // 2] * 1e6:7.1f} us "
              f"(min {ts[0] * 1e6:7.1f})  kernels {k * 1e6:7.1f} us", flush=True)
    m.free()
