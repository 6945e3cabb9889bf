"""Times band-major ELL SpMV variants (spmvtk_k_tune "ell_variant": 0 = LSU
loads, 1 = TMA bulk-copy ring 8 bands x 3 stages, 2 = 4 x 4) on BASELINE
configs and checks them against variant 0."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param, d in ((1, 256, 0.0), (2, 1 << 20, 0.0), (3, 128, 0.0), (5, 1 << 21, 0.0),
                      (5, 1 << 21, 0.5)):
    m = sp.HostCrs(cfg, param, d).upload()
    e = m.convert(sp.Format.ELL)
    dd = e.describe()
    n, nz = dd.n, dd.band_count
    x = torch.from_numpy(sp.gen_vector(n, 3)).cuda()
    y = torch.empty_like(x)
    ref = None
    for v in (0, 1, 2, 3, 4):
        lib.spmvtk_k_tune(b"ell_variant", v)
        for _ in range(5):
            e.spmv_device(sp.Kernel.ELL_INNER, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            e.spmv_device(sp.Kernel.ELL_INNER, x.data_ptr(), y.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 100 * 1e-3
        if ref is None:
            ref = y.clone()
        err = float(((y - ref).abs().max() / ref.abs().max()).item())
        print(f"cfg{cfg} D={d} nz={nz} ell v{v}: {t*1e6:8.1f} us "
              f"{(12*n*nz+16*n)/t/1e9:7.0f} GB/s err={err:.1e}", flush=True)
    lib.spmvtk_k_tune(b"ell_variant", 0)
    e.free()
    m.free()
