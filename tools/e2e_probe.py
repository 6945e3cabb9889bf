"""Diagnoses the e2e path: PCIe copy times and spmvtk_spmv breakdown."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

n = 1 << 20
xh = torch.empty(n, dtype=torch.float64).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda")


def t(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print("H2D 8MB pinned  ms", t(lambda: xd.copy_(xh, non_blocking=True)))
print("D2H 8MB pinned  ms", t(lambda: yh.copy_(xd, non_blocking=True)))
print("both, one stream ms", t(lambda: (xd.copy_(xh, non_blocking=True), yh.copy_(xd, non_blocking=True))))
# full duplex: the copy-in and the copy-out on their own streams
yd = torch.empty_like(xd)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def duplex():
    with torch.cuda.stream(s_in):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s_out):
        yh.copy_(yd, non_blocking=True)


print("both, two streams (duplex) ms", t(duplex))
lib = sp.load_library()
cudart = C.CDLL("libcudart.so.12") if False else None
m = sp.HostCrs(2, n).upload()
ell = m.convert(sp.Format.ELL)
xn, yn = xh.numpy(), yh.numpy()
for k, h in ((sp.Kernel.ELL_INNER, ell), (sp.Kernel.CRS, m)):
    print(k.name, "spmv pinned ms", t(lambda: h.spmv(xn, k, 1, out=yn)))
    xp, yp = np.empty(n), np.empty(n)
    print(k.name, "spmv pageable ms", t(lambda: h.spmv(xp, k, 1, out=yp)))
streams = [torch.cuda.Stream() for _ in range(4)]


def split_h2d(k):
    step = n // k
    cur = torch.cuda.current_stream()
    for i in range(k):
        s = streams[i]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            xd[i * step:(i + 1) * step].copy_(xh[i * step:(i + 1) * step], non_blocking=True)
    for i in range(k):
        cur.wait_stream(streams[i])


for k in (1, 2, 4):
    print(f"H2D split {k} ms", t(lambda: split_h2d(k)))
big = torch.empty(1 << 25, dtype=torch.float64).pin_memory()
bigd = torch.empty(1 << 25, dtype=torch.float64, device="cuda")
print("H2D 256MB GB/s", 256 * 2**20 / (t(lambda: bigd.copy_(big, non_blocking=True), 5) * 1e-3) / 1e9)
print("D2H 256MB GB/s", 256 * 2**20 / (t(lambda: big.copy_(bigd, non_blocking=True), 5) * 1e-3) / 1e9)
