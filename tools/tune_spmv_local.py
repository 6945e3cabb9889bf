"""SpMV kernel time with SM-local row regions (knob spmv_local = CTAs per SM,
0 = interleaved grid passes) on banded and random matrices; results compared
with the interleaved mapping (max-norm relative error).

    python tools/tune_spmv_local.py [--configs 5,3,2] [--dparams 0.0,0.5,1.0,2.0] [--ks 0,1,2,4,8]
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
ap.add_argument("--configs", default="5,3,2")
ap.add_argument("--dparams", default="0.0,0.5,1.0,2.0")
ap.add_argument("--ks", default="0,1,2,4,8")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--formats", default="crs,ell,ell-row")
ap.add_argument("--knob", default="spmv_local")
ap.add_argument("--ones", action="store_true", help="x = 1 (as measure_spmv) instead of U(-1,1)")
a = ap.parse_args()
lib = sp.load_library()
KNOB = a.knob.encode()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}
KIND = {"crs": (None, sp.Kernel.CRS), "ell": (sp.Format.ELL, sp.Kernel.ELL_INNER),
        "ell-row": (sp.Format.ELL_ROWMAJOR, sp.Kernel.ELL_ROWMAJOR)}
ks = [int(k) for k in a.ks.split(",")]
for cfg in [int(c) for c in a.configs.split(",")]:
    for dp in ([float(x) for x in a.dparams.split(",")] if cfg == 5 else [0.0]):
        m = sp.HostCrs(cfg, PARAM[cfg], dp).upload()
        d = m.describe()
        x = (torch.ones(d.n, dtype=torch.float64) if a.ones
             else torch.from_numpy(sp.gen_vector(d.n, 7))).cuda()
        y = torch.empty(d.n, dtype=torch.float64, device="cuda")
        for fname in a.formats.split(","):
            fmt, kern = KIND[fname]
            try:
                h = m if fmt is None else m.convert(fmt, max_bytes=40 << 30)
            except sp.SpmvtkError as e:
                print(f"cfg{cfg} D={dp} {fname}: {e.message}")
                continue
            line = f"cfg{cfg} D={dp} {fname:7s}:"
            ref = None
            for k in ks:
                lib.spmvtk_k_tune(KNOB, k)
                h.spmv_device(kern, x.data_ptr(), y.data_ptr())
                torch.cuda.synchronize()
                got = y.cpu().numpy().copy()
                if ref is None:
                    ref = got
                err = np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)
                for _ in range(3):
                    h.spmv_device(kern, x.data_ptr(), y.data_ptr())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(a.reps):
                    h.spmv_device(kern, x.data_ptr(), y.data_ptr())
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / a.reps * 1e3
                line += f"  k={k}: {t:7.1f} us" + ("" if err <= 1e-12 else f" ERR {err:.1e}")
            if fmt is None and a.knob == "spmv_local":  # the library's own measure_spmv (t_crs of the AT records)
                for k in ks:
                    lib.spmvtk_k_tune(KNOB, k)
                    line += f"  [measure_spmv k={k}: {sp.bench(m, sp.Kernel.COO_ROW_OUTER)['t_crs'] * 1e6:7.1f} us]"
            lib.spmvtk_k_tune(KNOB, 0)
            print(line, flush=True)
            if h is not m:
                h.free()
        m.free()
