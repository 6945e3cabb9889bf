"""Structured fuzzing of the whole path on the GPU against the C port.

Shapes the fixed fixtures do not reach: n = 1, 31/32/33 (warp edges),
empty matrices, all-empty rows, a single dense row or column (oversized
CCS buckets, long CRS rows), power-law and banded rows, duplicate-free
unsorted columns, sizes that cross the CCS two-pass and staged-partition
thresholds.  Every transform is bit-exact, every SpMV kernel within 1e-12 of
the port's sequential CRS product, and every handle converts back to the
canonical CRS.
"""
import zlib

import numpy as np
import pytest

from oracle.oracle import max_rel_error

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _rows_to_crs(n, rows, rng, shuffle):
    lens = np.array([len(r) for r in rows], np.int64)
    if shuffle:
        rows = [rng.permutation(r) for r in rows]
    ci = np.concatenate(rows).astype(np.int64) if lens.sum() else np.zeros(0, np.int64)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return rp + 1, ci + 1, rng.standard_normal(ci.shape[0])


def _case(kind, n, rng):
    if kind == "empty":
        rows = [np.zeros(0, np.int64) for _ in range(n)]
    elif kind == "diag":
        rows = [np.array([i]) for i in range(n)]
    elif kind == "random":
        rows = [np.sort(rng.choice(n, size=min(n, int(rng.integers(0, 12))), replace=False))
                for _ in range(n)]
    elif kind == "banded":
        rows = [np.arange(max(0, i - 3), min(n, i + 4)) for i in range(n)]
    elif kind == "dense_row":
        rows = [np.zeros(0, np.int64) for _ in range(n)]
        rows[n // 2] = np.arange(n)
        for i in range(0, n, 7):
            if i != n // 2:
                rows[i] = np.array([i])
    elif kind == "dense_col":
        rows = [np.unique(np.array([0, i, n - 1])) for i in range(n)]
    elif kind == "powerlaw":
        lens = np.minimum(n, np.round(rng.lognormal(1.5, 1.3, size=n)).astype(int))
        rows = [np.sort(rng.choice(n, size=int(ln), replace=False)) for ln in lens]
    else:
        raise ValueError(kind)
    return rows


CASES = [(k, n) for k in ("empty", "diag", "random", "banded") for n in (1, 2, 31, 32, 33, 257)]
CASES += [("dense_row", 3000), ("dense_col", 3000), ("powerlaw", 4000), ("random", 70000),
          ("banded", 70000), ("powerlaw", 70000), ("dense_col", 20000)]


@pytest.mark.parametrize("kind,n", CASES)
def test_fuzz_path(gpu, port, kind, n):
    sp = gpu
    rng = np.random.default_rng(zlib.crc32(f"{kind}:{n}".encode()))
    rows = _case(kind, n, rng)
    rp, ci, v = _rows_to_crs(n, rows, rng, shuffle=kind == "random")
    x = rng.uniform(-1, 1, n)
    m = sp.Matrix.from_crs(n, rp, ci, v, index_base=1)
    want = port.spmv_crs(n, rp, ci, v, x)
    # transforms, bit-exact
    cp, ri, cv = port.crs_to_ccs(n, rp, ci, v)
    ccs = m.convert(sp.Format.CCS)
    np.testing.assert_array_equal(ccs.array(sp.Array.POINTER, 8, 1), cp)
    np.testing.assert_array_equal(ccs.array(sp.Array.ROW_IDX, 8, 1), ri)
    assert ccs.array(sp.Array.VALUES).tobytes() == cv.tobytes()
    r, c, vv = port.crs_to_coo_row(n, rp, ci, v)
    coo = m.convert(sp.Format.COO_ROW)
    np.testing.assert_array_equal(coo.array(sp.Array.ROW_IDX, 8, 1), r)
    np.testing.assert_array_equal(coo.array(sp.Array.COL_IDX, 8, 1), c)
    assert coo.array(sp.Array.VALUES).tobytes() == vv.tobytes()
    cr, cc, cvv = port.crs_to_coo_col(n, rp, ci, v)
    cooc = m.convert(sp.Format.COO_COL)
    np.testing.assert_array_equal(cooc.array(sp.Array.ROW_IDX, 8, 1), cr)
    np.testing.assert_array_equal(cooc.array(sp.Array.COL_IDX, 8, 1), cc)
    assert cooc.array(sp.Array.VALUES).tobytes() == cvv.tobytes()
    bc, ev, ec, cnt = port.crs_to_ell(n, rp, ci, v)
    ell = m.convert(sp.Format.ELL)
    assert ell.describe().band_count == bc
    assert ell.array(sp.Array.VALUES).tobytes() == ev.tobytes()
    np.testing.assert_array_equal(ell.array(sp.Array.COL_IDX, 8, 1), ec)
    np.testing.assert_array_equal(ell.array(sp.Array.ROW_ENTRY_COUNT), cnt)
    rvals, rcols = port.ell_to_rowmajor(n, bc, ev, ec)
    ellr = m.convert(sp.Format.ELL_ROWMAJOR)
    assert ellr.array(sp.Array.VALUES).tobytes() == rvals.tobytes()
    np.testing.assert_array_equal(ellr.array(sp.Array.COL_IDX, 8, 1), rcols)
    # every SpMV kernel
    for h, k in ((m, sp.Kernel.CRS), (coo, sp.Kernel.COO_ROW_OUTER),
                 (cooc, sp.Kernel.COO_COL_OUTER), (ell, sp.Kernel.ELL_INNER),
                 (ell, sp.Kernel.ELL_OUTER), (ellr, sp.Kernel.ELL_ROWMAJOR)):
        y, _ = h.spmv(x, k, lanes=3)
        assert max_rel_error(y, want) <= TOL, (kind, n, k)
    # back to the canonical CRS from every handle
    crp = rp
    order = (np.concatenate([np.argsort(ci[crp[i] - 1:crp[i + 1] - 1], kind="stable") +
                             crp[i] - 1 for i in range(n)]).astype(np.int64)
             if v.size else np.zeros(0, np.int64))
    for h in (ccs, coo, cooc, ell, ellr):
        back = h.to_crs()
        np.testing.assert_array_equal(back.array(sp.Array.POINTER, 8, 1), crp)
        np.testing.assert_array_equal(back.array(sp.Array.COL_IDX, 8, 1), ci[order])
        assert back.array(sp.Array.VALUES).tobytes() == v[order].tobytes()
        back.free()
    for h in (ccs, coo, cooc, ell, ellr, m):
        h.free()


STABLE_CASES = [("random", 33), ("random", 257), ("banded", 70000), ("powerlaw", 70000),
                ("dense_col", 20000), ("dense_row", 3000), ("empty", 32), ("diag", 1)]


@pytest.mark.parametrize("kind,n", STABLE_CASES)
def test_stable_ccs_pipeline(gpu, port, kind, n):
    """The stable partition pipeline (kernels_ccs.cu), forced for matrices the
    rank-by-row pipeline would take, is bit-exact against the port too."""
    sp = gpu
    lib = sp.load_library()
    rng = np.random.default_rng(zlib.crc32(f"stable:{kind}:{n}".encode()))
    rows = _case(kind, n, rng)
    rp, ci, v = _rows_to_crs(n, rows, rng, shuffle=kind == "random")
    m = sp.Matrix.from_crs(n, rp, ci, v, index_base=1)
    assert lib.spmvtk_k_tune(b"ccs_stable", 1) == 0
    try:
        cp, ri, cv = port.crs_to_ccs(n, rp, ci, v)
        ccs = m.convert(sp.Format.CCS)
        np.testing.assert_array_equal(ccs.array(sp.Array.POINTER, 8, 1), cp)
        np.testing.assert_array_equal(ccs.array(sp.Array.ROW_IDX, 8, 1), ri)
        assert ccs.array(sp.Array.VALUES).tobytes() == cv.tobytes()
        cr, cc, cvv = port.crs_to_coo_col(n, rp, ci, v)
        cooc = m.convert(sp.Format.COO_COL)
        np.testing.assert_array_equal(cooc.array(sp.Array.ROW_IDX, 8, 1), cr)
        np.testing.assert_array_equal(cooc.array(sp.Array.COL_IDX, 8, 1), cc)
        assert cooc.array(sp.Array.VALUES).tobytes() == cvv.tobytes()
        for h in (ccs, cooc):
            h.free()
    finally:
        lib.spmvtk_k_tune(b"ccs_stable", 0)
        m.free()


@pytest.mark.parametrize("n,dups", [(50, 40), (3000, 2500), (70000, 50000)])
def test_ccs_with_duplicate_pairs(gpu, port, n, dups):
    """A CRS holding duplicate (row, col) pairs (allowed by crs_to_ccs,
    convert.cpp:24-53): the conversion keeps every copy in CRS order, exactly
    as the reference's cursor scatter -- routed to the stable pipeline by the
    handle's ordering check."""
    sp = gpu
    rng = np.random.default_rng(n)
    rows = [np.sort(rng.choice(n, size=int(rng.integers(0, 6)), replace=False)) for _ in range(n)]
    for i in rng.choice(n, size=dups):  # repeat one of the row's columns
        if rows[i].size:
            rows[i] = np.sort(np.append(rows[i], rows[i][rng.integers(0, rows[i].size)]))
    rp, ci, v = _rows_to_crs(n, rows, rng, shuffle=False)
    m = sp.Matrix.from_crs(n, rp, ci, v, index_base=1)
    cp, ri, cv = port.crs_to_ccs(n, rp, ci, v)
    ccs = m.convert(sp.Format.CCS)
    np.testing.assert_array_equal(ccs.array(sp.Array.POINTER, 8, 1), cp)
    np.testing.assert_array_equal(ccs.array(sp.Array.ROW_IDX, 8, 1), ri)
    assert ccs.array(sp.Array.VALUES).tobytes() == cv.tobytes()
    cr, cc, cvv = port.crs_to_coo_col(n, rp, ci, v)
    cooc = m.convert(sp.Format.COO_COL)
    np.testing.assert_array_equal(cooc.array(sp.Array.ROW_IDX, 8, 1), cr)
    np.testing.assert_array_equal(cooc.array(sp.Array.COL_IDX, 8, 1), cc)
    assert cooc.array(sp.Array.VALUES).tobytes() == cvv.tobytes()
    for h in (ccs, cooc, m):
        h.free()
