"""Breaks down t_trans of CRS->ELL (config 2): wall clock of the public
convert call vs the row-statistics round trip alone vs the kernels alone."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

sp.set_stream(torch.cuda.current_stream().cuda_stream)
sp.reserve_device_memory(8 << 30)
m = sp.HostCrs(2, 1 << 20).upload()
for _ in range(3):
    m.convert(sp.Format.ELL).free()


def wall(fn, reps=20):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        if r is not None and hasattr(r, "free"):
            r.free()
    ts.sort()
    return ts[len(ts) // 2] * 1e6


print(f"convert(ELL) wall      {wall(lambda: m.convert(sp.Format.ELL)):8.1f} us")
print(f"row_stats() wall       {wall(lambda: m.row_stats()):8.1f} us")
print(f"empty sync wall        {wall(lambda: None):8.1f} us")
print(f"ELL kernels (events)   {m.transform_kernel_seconds(sp.Format.ELL, 15) * 1e6:8.1f} us")
print(f"convert(COO_ROW) wall  {wall(lambda: m.convert(sp.Format.COO_ROW)):8.1f} us")
print(f"COO_ROW kernel         {m.transform_kernel_seconds(sp.Format.COO_ROW, 15) * 1e6:8.1f} us")
