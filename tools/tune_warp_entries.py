"""CRS->COO-row with 512 / 1024 / 2048 entries per warp chunk."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param in ((2, 1 << 20), (3, 128), (4, 1 << 22), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    for we in (256, 128, 512, 1024):
        lib.spmvtk_k_tune(b"warp_entries", we)
        t = m.transform_kernel_seconds(sp.Format.COO_ROW, 9)
        print(f"cfg{cfg} warp_entries={we}: coo-row {t*1e6:8.1f} us", flush=True)
    lib.spmvtk_k_tune(b"warp_entries", 512)
    m.free()
