"""Streaming host SpMV: ms per product with SPMVTK_PIPE_SPLIT copy streams per direction
and SPMVTK_PIPE_SLOTS products in flight (host time of the submits printed too)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2407_00019_b200 import spmvtk as sp
m = sp.HostCrs(2, 1 << 20).upload(); e = m.convert(sp.Format.ELL); n = m.describe().n
xs = [torch.from_numpy(sp.gen_vector(n, 1 + i)).pin_memory() for i in range(2)]
ys = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
pipe = sp.Pipeline(e, sp.Kernel.ELL_INNER)
for i in range(4): pipe.submit(xs[i % 2].numpy(), ys[i % 2].numpy())
pipe.wait()
t0 = time.perf_counter()
for i in range(200): pipe.submit(xs[i % 2].numpy(), ys[i % 2].numpy())
t1 = time.perf_counter()
pipe.wait()
print("split", os.environ.get("SPMVTK_PIPE_SPLIT", "2"), "slots", os.environ.get("SPMVTK_PIPE_SLOTS", "3"),
      "ms/step", (time.perf_counter() - t0) / 200 * 1e3, "submit ms", (t1 - t0) / 200 * 1e3, flush=True)
