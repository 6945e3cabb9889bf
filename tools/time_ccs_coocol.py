"""Kernel time of CRS->CCS and CRS->COO-col (Phase I with the fused Phase II) on configs 2-5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_00019_b200 import spmvtk as sp
sp.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, param in ((2, 1 << 20), (3, 128), (4, 1 << 22), (5, 1 << 21)):
    m = sp.HostCrs(cfg, param).upload()
    a = m.transform_kernel_seconds(sp.Format.CCS, 15)
    b = m.transform_kernel_seconds(sp.Format.COO_COL, 15)
    print(f"cfg{cfg} ccs {a*1e6:8.1f} us  coo-col {b*1e6:8.1f} us", flush=True)
    m.free()
