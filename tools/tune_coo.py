"""Times COO-row / COO-col SpMV on configs 2, 3, 5 (GB/s of 16 nnz + 16 n)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param in ((2, 1 << 20), (3, 128), (4, 1 << 22), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    d = m.describe()
    x = torch.ones(d.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for name, fmt, k in (("coo-row", sp.Format.COO_ROW, sp.Kernel.COO_ROW_OUTER),
                         ("coo-col", sp.Format.COO_COL, sp.Kernel.COO_COL_OUTER)):
        h = m.convert(fmt)
        for _ in range(5):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 100 * 1e-3
        print(f"cfg{cfg} {name}: {t*1e6:8.1f} us {(16*d.nnz+16*d.n)/t/1e9:7.0f} GB/s", flush=True)
        h.free()
    m.free()
