"""Times the bucketed CRS->CCS kernels for several (coarse, sort threads)
settings.  coarse = log2 of the coarse bucket target of the two-pass
partition (0 = single pass)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

lib = sp.load_library()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
SETTINGS = [(9, 148, 1024, 0), (9, 148, 1024, 1)]
for cfg, param in ((2, 1 << 20), (3, 128), (4, 1 << 22), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    for coarse, ns, stt, wnd in SETTINGS:
        lib.spmvtk_k_tune(b"ccs_window", wnd)
        lib.spmvtk_k_tune(b"ccs_coarse", coarse)
        lib.spmvtk_k_tune(b"ccs_slices", ns)
        lib.spmvtk_k_tune(b"ccs_stage_threads", stt)
        t = m.transform_kernel_seconds(sp.Format.CCS, 15)
        print(f"cfg{cfg} coarse={coarse} slices={ns} stage_threads={stt} window={wnd}: "
              f"{t*1e6:8.1f} us",
              flush=True)
    lib.spmvtk_k_tune(b"ccs_slices", 148)
    lib.spmvtk_k_tune(b"ccs_stage_threads", 1024)
    lib.spmvtk_k_tune(b"ccs_window", 1)
    m.free()
