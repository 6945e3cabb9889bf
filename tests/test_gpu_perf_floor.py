"""Loose throughput floors for the SpMV kernels on the BASELINE workloads.

Not a benchmark (bench.py is): a regression tripwire.  The floors sit about
30% under the rates measured on B200 (profiles/r01_tune_*),
so a clock dip does not trip them but a kernel that loses its 128-bit loads
or falls back to a slower variant does (a 64-bit induction-variable change
once cost the stencil CRS kernel 40% unnoticed).
"""
import pytest

pytestmark = pytest.mark.gpu

# (config, param, format, kernel name, GB/s floor)
FLOORS = [
    (2, 1 << 20, "crs", "CRS", 1700.0),
    (2, 1 << 20, "ell", "ELL_INNER", 2800.0),
    (2, 1 << 20, "coo-row", "COO_ROW_OUTER", 1900.0),
    (3, 128, "crs", "CRS", 3700.0),
    (3, 128, "ell", "ELL_INNER", 4800.0),
    (3, 128, "ell-row", "ELL_ROWMAJOR", 3400.0),
]


def _time(fn, torch, reps=100):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


@pytest.mark.parametrize("cfg", [2, 3])
def test_spmv_throughput_floors(gpu, cfg):
    import torch
    sp = gpu
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    rows = [f for f in FLOORS if f[0] == cfg]
    m = sp.HostCrs(cfg, rows[0][1]).upload()
    d = m.describe()
    n, nnz = d.n, d.nnz
    fmts = {"crs": None, "ell": sp.Format.ELL, "coo-row": sp.Format.COO_ROW,
            "ell-row": sp.Format.ELL_ROWMAJOR}
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    failures = []
    for _, _, fmt, kname, floor in rows:
        h = m if fmts[fmt] is None else m.convert(fmts[fmt])
        k = getattr(sp.Kernel, kname)
        t = _time(lambda: h.spmv_device(k, x.data_ptr(), y.data_ptr()), torch)
        if fmt == "crs":
            nbytes = 12 * nnz + 4 * (n + 1) + 16 * n
        elif fmt == "coo-row":
            nbytes = 16 * nnz + 16 * n
        else:
            nbytes = 12 * n * h.describe().band_count + 16 * n
        gbs = nbytes / t / 1e9
        if gbs < floor:
            failures.append(f"cfg{cfg} {fmt}: {gbs:.0f} GB/s < floor {floor:.0f}")
        if h is not m:
            h.free()
    m.free()
    assert not failures, failures
