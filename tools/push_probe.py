"""Per-launch cost of the pushed CRS SpMV pieces on one GPU (config 4):
plain y store, push store (1 destination), + sparse mask, + flag wait /
counter / signal, two destinations; the same for ELL.  CUDA events on the current stream, median of 20."""
import ctypes as C
import json

import torch

from paper_2407_00019_b200 import spmvtk as sp


def timed(fn, reps=20):
    for _ in range(3):
        fn(0)
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(i + 3)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    torch.cuda.set_device(0)
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    h = sp.HostCrs(4, 4194304, 0.0, 2407)
    m = h.upload()
    n = m.describe().n
    x = torch.from_numpy(sp.gen_vector(n, 1)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    mask = torch.ones(n, dtype=torch.uint8, device="cuda")
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = {"plain": timed(lambda i: m.spmv_device(sp.Kernel.CRS, x.data_ptr(), y.data_ptr()))}
    p = sp.Push()
    p.dst[0] = y.data_ptr()
    p.ndst = 1
    out["push_1dst"] = timed(lambda i: m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), p))
    pm = sp.Push()
    pm.dst[0] = y.data_ptr()
    pm.ndst = 1
    pm.mask = mask.data_ptr()
    out["push_mask"] = timed(lambda i: m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), pm))

    def synced(i):
        s = sp.PushSync()
        s.wait_flags = flags.data_ptr()
        s.nwait = 1
        s.wait_value = 0
        s.timeout_ns = 10**10
        s.status = status.data_ptr()
        s.signal.ptr[0] = flags.data_ptr()
        s.signal.n = 1
        s.signal_value = 0
        s.counter = counter.data_ptr()
        m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), pm, s)
    out["push_mask_sync"] = timed(synced)
    # two destinations (both on this GPU): the staged tile copy
    y2 = torch.empty(n, dtype=torch.float64, device="cuda")
    p2 = sp.Push()
    p2.dst[0], p2.dst[1] = y.data_ptr(), y2.data_ptr()
    p2.ndst = 2
    out["push_2dst"] = timed(lambda i: m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), p2))
    torch.testing.assert_close(y, y2, rtol=0, atol=0)
    # ELL on config 2 (config 4's padded ELL does not fit)
    m.free()
    m = sp.HostCrs(2, 1 << 20, 0.0, 2407).upload()
    n = m.describe().n
    x = torch.from_numpy(sp.gen_vector(n, 1)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    y2 = torch.empty(n, dtype=torch.float64, device="cuda")
    p.dst[0] = p2.dst[0] = y.data_ptr()
    p2.dst[1] = y2.data_ptr()
    out["c2_crs_plain"] = timed(lambda i: m.spmv_device(sp.Kernel.CRS, x.data_ptr(), y.data_ptr()))
    out["c2_crs_push_1dst"] = timed(lambda i: m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), p))
    e = m.convert(sp.Format.ELL)
    out["ell_plain"] = timed(lambda i: e.spmv_device(sp.Kernel.ELL_INNER, x.data_ptr(), y.data_ptr()))
    out["ell_push_1dst"] = timed(lambda i: e.spmv_device_push(sp.Kernel.ELL_INNER, x.data_ptr(), p))
    out["ell_push_2dst"] = timed(lambda i: e.spmv_device_push(sp.Kernel.ELL_INNER, x.data_ptr(), p2))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
