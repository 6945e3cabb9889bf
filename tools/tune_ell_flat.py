"""Times CRS->ELL (band-major, nz <= 32): auto (256-row CTAs for nz <= 8), 64- and 128-row CTAs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param in ((1, 256), (2, 1 << 20), (3, 128), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    for rows in (0, 64, 128):
        lib.spmvtk_k_tune(b"ell_flat_rows", rows)
        for fmt in (sp.Format.ELL,):
            t = m.transform_kernel_seconds(fmt, 9)
            print(f"cfg{cfg} rows={rows} {fmt.name}: {t*1e6:8.1f} us", flush=True)
    m.free()
lib.spmvtk_k_tune(b"ell_flat_rows", 0)
