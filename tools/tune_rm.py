"""Times row-major ELL SpMV variants (spmvtk_k_tune("rm_variant", v)).

    python tools/tune_rm.py [-1,12,16,...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param in ((2, 1 << 20), (3, 128), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    d = m.describe()
    nz = m.row_stats().max_row
    e = m.convert(sp.Format.ELL_ROWMAJOR)
    x = torch.rand(d.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    b = 12 * d.n * nz + 16 * d.n
    for v in [int(t) for t in (sys.argv[1] if len(sys.argv) > 1 else "-1,12,16,17,18,21,22,23,24").split(",")]:
        lib.spmvtk_k_tune(b"rm_variant", v)
        for _ in range(5):
            e.spmv_device(sp.Kernel.ELL_ROWMAJOR, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            e.spmv_device(sp.Kernel.ELL_ROWMAJOR, x.data_ptr(), y.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 100 * 1e-3
        print(f"cfg{cfg} nz={nz} rm v{v}: {t*1e6:7.1f} us {b/t/1e9:6.0f} GB/s", flush=True)
    lib.spmvtk_k_tune(b"rm_variant", -1)
