"""Guard-zone checks of every SpMV kernel (compute-sanitizer is closed on
this pool, so out-of-bounds accesses are caught by construction instead):
x sits inside a buffer whose guard zones hold NaN -- any gather outside
[0, ncols) poisons y -- and y inside a buffer whose guard zones hold a
sentinel that must survive -- any store outside [0, n) overwrites it.  The
structured fuzz shapes of test_gpu_fuzz.py (warp edges, empty rows, a dense
row / column, power-law rows) plus a row-block shard with ncols > rows.
"""
import zlib

import numpy as np
import pytest

from oracle.oracle import max_rel_error
from test_gpu_fuzz import _case, _rows_to_crs

pytestmark = pytest.mark.gpu
G = 4096  # guard elements on each side
SENTINEL = 7.77e300

SHAPES = [("empty", 33), ("diag", 1), ("random", 31), ("random", 257), ("banded", 2000),
          ("dense_row", 3000), ("dense_col", 3000), ("powerlaw", 4000), ("powerlaw", 70000)]


def _guarded_spmv(torch, h, k, x, n_out):
    xb = torch.full((x.shape[0] + 2 * G,), float("nan"), dtype=torch.float64, device="cuda")
    xb[G:G + x.shape[0]] = torch.from_numpy(x).cuda()
    yb = torch.full((n_out + 2 * G,), SENTINEL, dtype=torch.float64, device="cuda")
    h.spmv_device(k, xb.data_ptr() + 8 * G, yb.data_ptr() + 8 * G)
    torch.cuda.synchronize()
    y = yb.cpu().numpy()
    assert np.all(y[:G] == SENTINEL) and np.all(y[G + n_out:] == SENTINEL), "store outside y"
    out = y[G:G + n_out]
    assert not np.any(np.isnan(out)), "gather outside x"
    return out


@pytest.mark.parametrize("kind,n", SHAPES)
def test_spmv_kernels_stay_inside_x_and_y(gpu, port, kind, n):
    import torch
    sp = gpu
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    rng = np.random.default_rng(zlib.crc32(f"guard:{kind}:{n}".encode()))
    rows = _case(kind, n, rng)
    rp, ci, v = _rows_to_crs(n, rows, rng, shuffle=kind == "random")
    x = rng.uniform(-1, 1, n)
    want = port.spmv_crs(n, rp, ci, v, x)
    m = sp.Matrix.from_crs(n, rp, ci, v, index_base=1)
    handles = [(m, sp.Kernel.CRS)]
    for fmt, k in ((sp.Format.COO_ROW, sp.Kernel.COO_ROW_OUTER),
                   (sp.Format.COO_COL, sp.Kernel.COO_COL_OUTER),
                   (sp.Format.ELL, sp.Kernel.ELL_INNER), (sp.Format.ELL, sp.Kernel.ELL_OUTER),
                   (sp.Format.ELL_ROWMAJOR, sp.Kernel.ELL_ROWMAJOR)):
        handles.append((m.convert(fmt), k))
    for h, k in handles:
        y = _guarded_spmv(torch, h, k, x, n)
        assert max_rel_error(y, want) <= 1e-12, (kind, n, k)
    # the CRS kernel variants, each forced
    lib = sp.load_library()
    for variant in (12, 16, 17, 18, 20, 21, 22):
        assert lib.spmvtk_k_tune(b"crs_variant", variant) == 0
        try:
            y = _guarded_spmv(torch, m, sp.Kernel.CRS, x, n)
        finally:
            lib.spmvtk_k_tune(b"crs_variant", -1)
        assert max_rel_error(y, want) <= 1e-12, (kind, n, variant)
    # the SM-local band-major ELL kernel (banded matrices), forced: bitwise
    # the default ELL kernel's result (same per-row band order)
    ell = handles[3][0]
    y_def = _guarded_spmv(torch, ell, sp.Kernel.ELL_INNER, x, n)
    assert lib.spmvtk_k_tune(b"ell_banded", 1) == 0
    try:
        y_loc = _guarded_spmv(torch, ell, sp.Kernel.ELL_INNER, x, n)
    finally:
        lib.spmvtk_k_tune(b"ell_banded", -1)
    assert y_loc.tobytes() == y_def.tobytes(), (kind, n, "ell_banded")
    # the row-major ELL variants (the sub-warp kernels on fixed-stride rows)
    rm = handles[-1][0]
    for variant in (12, 16, 17, 18, 21, 22):
        assert lib.spmvtk_k_tune(b"rm_variant", variant) == 0
        try:
            y = _guarded_spmv(torch, rm, sp.Kernel.ELL_ROWMAJOR, x, n)
        finally:
            lib.spmvtk_k_tune(b"rm_variant", -1)
        assert max_rel_error(y, want) <= 1e-12, (kind, n, "rm", variant)
    for h, _ in handles[1:]:
        h.free()
    m.free()


def test_shard_kernels_stay_inside_x_and_y(gpu, port):
    """A row-block shard reads global columns [0, ncols) and writes its own
    rows only (the multi-GPU layout)."""
    import torch
    sp = gpu
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    full = sp.HostCrs(4, 20000, 0.0, 3)
    rp, ci, v = full.arrays(1)
    n = full.n
    x = sp.gen_vector(n, 5)
    want = port.spmv_crs(n, rp, ci, v, x)
    for rank in range(3):
        h = sp.gen_baseline_shard_host(4, 20000, 0.0, 3, rank, 3)
        shard = h.upload()
        d = shard.describe()
        assert d.ncols == n and d.n < n
        for hh, k in ((shard, sp.Kernel.CRS), (shard.convert(sp.Format.ELL), sp.Kernel.ELL_INNER),
                      (shard.convert(sp.Format.COO_ROW), sp.Kernel.COO_ROW_OUTER)):
            y = _guarded_spmv(torch, hh, k, x, d.n)
            assert max_rel_error(y, want[d.row_offset:d.row_offset + d.n]) <= 1e-12
            if hh is not shard:
                hh.free()
        shard.free()
        h.free()
