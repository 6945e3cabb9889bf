"""COO-row SpMV: entries per warp (spmvtk_k_tune "coo_chunk"; 0 = automatic)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2407_00019_b200 import spmvtk as sp
lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param in ((2, 1 << 20), (3, 128), (4, 1 << 22), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    d = m.describe()
    h = m.convert(sp.Format.COO_ROW)
    x = torch.ones(d.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    for ch in (0, 2048, 1024):
        lib.spmvtk_k_tune(b"coo_chunk", ch)
        for _ in range(5): h.spmv_device(sp.Kernel.COO_ROW_OUTER, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100): h.spmv_device(sp.Kernel.COO_ROW_OUTER, x.data_ptr(), y.data_ptr())
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 100 * 1e-3
        print(f"cfg{cfg} chunk={ch}: {t*1e6:8.1f} us {(16*d.nnz+16*d.n)/t/1e9:7.0f} GB/s", flush=True)
    h.free(); m.free()
