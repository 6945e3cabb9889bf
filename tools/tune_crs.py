"""Times kernel variants (spmvtk_k_tune knobs) on the BASELINE workloads and
prints GB/s of the compulsory bytes.  Tuning aid only, not a bench.

    python tools/tune_crs.py "2:1048576,3:128" "0,8,13" [hint-values] [ell]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
configs = [(int(c.split(":")[0]), int(c.split(":")[1])) for c in
           (sys.argv[1] if len(sys.argv) > 1 else "2:1048576,3:128,1:256,4:4194304").split(",")]
variants = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,8,13").split(",")]
hints = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "0,1").split(",")]
do_ell = len(sys.argv) > 4 and sys.argv[4] == "ell"


def timeit(fn, reps=200):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


for cfg, param in configs:
    m = sp.HostCrs(cfg, param).upload()
    d = m.describe()
    st = m.row_stats()
    n, nnz = d.n, d.nnz
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    byts = 12 * nnz + 4 * (n + 1) + 16 * n
    print(f"config {cfg} n={n} nnz={nnz} mean={nnz/n:.1f} max_row={st.max_row} "
          f"d_mat={st.d_mat:.4f}", flush=True)
    ref = None
    for h in hints:
        lib.spmvtk_k_tune(b"l2_hint", h)
        for v in variants:
            lib.spmvtk_k_tune(b"crs_variant", v)
            t = timeit(lambda: m.spmv_device(sp.Kernel.CRS, x.data_ptr(), y.data_ptr()))
            yy = y.cpu().numpy()
            if ref is None:
                ref = yy
            err = float(np.max(np.abs(yy - ref)) / max(1e-300, np.max(np.abs(ref))))
            print(f"    crs v{v} hint={h}: {t*1e6:8.1f} us {byts/t/1e9:7.0f} GB/s err={err:.1e}",
                  flush=True)
        if do_ell and st.max_row <= 64:
            ell = m.convert(sp.Format.ELL)
            eb = 12 * n * st.max_row + 16 * n
            t = timeit(lambda: ell.spmv_device(sp.Kernel.ELL_INNER, x.data_ptr(), y.data_ptr()))
            print(f"    ell-inner hint={h}: {t*1e6:8.1f} us {eb/t/1e9:7.0f} GB/s", flush=True)
            ell.free()
    lib.spmvtk_k_tune(b"crs_variant", -1)
    lib.spmvtk_k_tune(b"l2_hint", 0)
    m.free()
