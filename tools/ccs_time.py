import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2407_00019_b200 import spmvtk as sp
sp.set_stream(torch.cuda.current_stream().cuda_stream)
PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}
for cfg, dp in ((1,0.0),(2,0.0),(3,0.0),(4,0.0),(5,0.0),(5,1.0),(5,2.0)):
    m = sp.HostCrs(cfg, PARAM[cfg], dp).upload()
    d = m.describe()
    for fmt in (sp.Format.CCS, sp.Format.COO_COL):
        t = m.transform_kernel_seconds(fmt, 10)
        print(f"cfg{cfg} D={dp} {fmt.name:8s} {t*1e6:9.1f} us  {(28*d.nnz+12*d.n)/t/1e9:6.0f} GB/s", flush=True)
    m.free()
