"""One CRS->ELL conversion of a BASELINE config (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

cfg = int(sys.argv[1])
fmt = sp.Format[sys.argv[2]] if len(sys.argv) > 2 else sp.Format.ELL
sp.set_stream(torch.cuda.current_stream().cuda_stream)
m = sp.HostCrs(cfg, {1: 256, 2: 1 << 20, 3: 128}[cfg]).upload()
torch.cuda.synchronize()
for _ in range(3):
    m.convert(fmt).free()
torch.cuda.synchronize()
print("ok")
