"""Parity of the CUDA path with the oracle, through the C ABI (GPU).

Transforms must be bit-exact against the reference (values memcmp, every
index equal after widening to the reference's 1-based int64); SpMV within
1e-12 max-norm relative of the reference (test_support.hpp:96-105; the
tolerance of BASELINE.json north_star), and within 1e-10 of a dense mat-vec.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle.oracle import dense_matvec, max_rel_error, random_crs

pytestmark = pytest.mark.gpu

TOL = 1e-12


def upload(sp, n, rp, ci, v):
    return sp.Matrix.from_crs(n, np.asarray(rp, np.int64), np.asarray(ci, np.int64),
                              np.asarray(v, np.float64), index_base=1)


def ref_layout(m, sp, which):
    return m.array(which, index_width=8, index_base=1)


# ---------------------------------------------------------------- KATs
def test_kat_transforms(gpu, kat):
    sp = gpu
    for c in kat["coo_row"]:
        m = upload(sp, c["n"], c["row_ptr"], c["col_idx"], c["values"])
        coo = m.convert(sp.Format.COO_ROW)
        assert coo.format == sp.Format.COO_ROW
        assert ref_layout(coo, sp, sp.Array.ROW_IDX).tolist() == c["row_idx"], c["ref"]
        assert ref_layout(coo, sp, sp.Array.COL_IDX).tolist() == c["out_col_idx"]
        assert coo.array(sp.Array.VALUES).tolist() == c["out_values"]
    for c in kat["ccs"]:
        m = upload(sp, c["n"], c["row_ptr"], c["col_idx"], c["values"])
        ccs = m.convert(sp.Format.CCS)
        assert ref_layout(ccs, sp, sp.Array.POINTER).tolist() == c["col_ptr"], c["ref"]
        assert ref_layout(ccs, sp, sp.Array.ROW_IDX).tolist() == c["row_idx"]
        assert ccs.array(sp.Array.VALUES).tolist() == c["out_values"]
    for c in kat["coo_col"]:
        m = upload(sp, c["n"], c["row_ptr"], c["col_idx"], c["values"])
        coo = m.convert(sp.Format.COO_COL)
        assert coo.format == sp.Format.COO_COL
        assert ref_layout(coo, sp, sp.Array.COL_IDX).tolist() == c["out_col_idx"], c["ref"]
        assert ref_layout(coo, sp, sp.Array.ROW_IDX).tolist() == c["row_idx"]
        assert coo.array(sp.Array.VALUES).tolist() == c["out_values"]
    for c in kat["ell"]:
        m = upload(sp, c["n"], c["row_ptr"], c["col_idx"], c["values"])
        ell = m.convert(sp.Format.ELL)
        d = ell.describe()
        assert d.band_count == c["band_count"] and d.nnz == c["stored_nnz"], c["ref"]
        # counts are not indices: exported as-is whatever the index base
        assert ref_layout(ell, sp, sp.Array.ROW_ENTRY_COUNT).tolist() == c["row_entry_count"]
        assert ell.array(sp.Array.ROW_ENTRY_COUNT, 4, 0).tolist() == c["row_entry_count"]
        if "out_values" in c:
            assert ell.array(sp.Array.VALUES).tolist() == c["out_values"]
            assert ref_layout(ell, sp, sp.Array.COL_IDX).tolist() == c["out_col_idx"]


def test_kat_guard_and_estimates(gpu, kat):
    sp = gpu
    g = kat["ell_guard"]
    n = g["n"]
    rp = np.full(n + 1, g["heavy_row_entries"] + 1, np.int64)
    rp[0] = 1
    ci = np.arange(1, g["heavy_row_entries"] + 1)
    m = upload(sp, n, rp, ci, np.ones(ci.shape[0]))
    for fmt in (sp.Format.ELL, sp.Format.ELL_ROWMAJOR):
        with pytest.raises(sp.SpmvtkError) as e:
            m.convert(fmt, max_bytes=g["max_bytes"])
        assert e.value.status == g["status"]
        assert g["message_contains"] in e.value.message
    assert m.info().ell_bytes == n * g["heavy_row_entries"] * 16
    # unlimited: the conversion goes through on the GPU
    ell = m.convert(sp.Format.ELL)
    assert ell.describe().band_count == g["heavy_row_entries"]
    c = kat["capi_guard"]
    heavy = sp.Matrix.gen_skewed(*c["gen_skewed"])
    with pytest.raises(sp.SpmvtkError) as e:
        heavy.convert(sp.Format.ELL, c["max_bytes"])
    assert e.value.status == sp.Status.ERR_MEMORY_LIMIT


def test_kat_spmv(gpu, kat):
    sp = gpu
    for c in kat["spmv_crs"]:
        m = upload(sp, c["n"], c["row_ptr"], c["col_idx"], c["values"])
        y, _ = m.spmv(c["x"], sp.Kernel.CRS)
        assert y.tolist() == c["y"], c["ref"]
    c = kat["spmv_dim_mismatch"]
    m = upload(sp, 2, [1, 1, 1], [], [])
    with pytest.raises(sp.SpmvtkError) as e:
        m.spmv(np.ones(c["x_len"]), sp.Kernel.CRS)
    assert e.value.status == c["status"]
    c = kat["ell_padding_spmv"]
    m = upload(sp, c["n"], c["row_ptr"], c["col_idx"], c["values"])
    for k, f in ((sp.Kernel.ELL_INNER, sp.Format.ELL), (sp.Kernel.ELL_OUTER, sp.Format.ELL),
                 (sp.Kernel.ELL_ROWMAJOR, sp.Format.ELL_ROWMAJOR)):
        y, _ = m.convert(f).spmv(c["x"], k)
        assert y.tolist() == c["y"]
    c = kat["ell_outer_idle_lanes"]
    n = c["n"]
    ident = upload(sp, n, np.arange(1, n + 2), np.arange(1, n + 1), np.ones(n))
    y, _ = ident.convert(sp.Format.ELL).spmv(c["x"], sp.Kernel.ELL_OUTER, lanes=c["lanes"])
    assert y.tolist() == c["y"]


def test_kat_ordering_contract(gpu, kat):
    sp = gpu
    c = kat["coo_ordering"]
    n = c["n"]
    ident = upload(sp, n, np.arange(1, n + 2), np.arange(1, n + 1), np.ones(n))
    coo_r = ident.convert(sp.Format.COO_ROW)
    with pytest.raises(sp.SpmvtkError) as e:
        coo_r.spmv(c["x"], sp.Kernel.COO_COL_OUTER, lanes=2)
    assert e.value.status == c["wrong_kernel_status"]
    assert "ordering" in e.value.message
    y, _ = coo_r.spmv(c["x"], sp.Kernel.COO_ROW_OUTER, lanes=2)
    assert y.tolist() == c["x"]
    with pytest.raises(sp.SpmvtkError) as e:
        coo_r.spmv(c["x"], sp.Kernel.ELL_INNER)
    assert e.value.status == sp.Status.ERR_USAGE
    with pytest.raises(sp.SpmvtkError) as e:
        coo_r.spmv(c["x"], sp.Kernel.COO_ROW_OUTER, lanes=0)
    assert e.value.status == sp.Status.ERR_USAGE


def test_kat_stats(gpu, kat):
    sp = gpu
    for c in kat["stats"]:
        counts = np.array(c["counts"], np.int64)
        n = len(counts)
        rp = np.concatenate([[1], 1 + np.cumsum(counts)])
        # statistics are structure-only; column 1 everywhere keeps indices in
        # range for any histogram (positions are not checked for distinctness)
        ci = np.ones(int(counts.sum()), np.int64)
        m = upload(sp, n, rp, ci, np.ones(ci.shape[0]))
        s = m.row_stats()
        if c.get("exact"):
            assert s.d_mat == c["d_mat"], c["ref"]
            if "mu" in c:
                assert s.mu == c["mu"] and s.sigma == c["sigma"]
        elif "d_mat" in c:
            assert s.mu == c["mu"] and s.sigma == c["sigma"] and s.d_mat == c["d_mat"]
        if c.get("d_mat_positive"):
            assert s.d_mat > 0
    c = kat["stats_empty"]
    m = upload(sp, c["n"], c["row_ptr"], [], [])
    with pytest.raises(sp.SpmvtkError) as e:
        m.info()
    assert e.value.status == c["status"]


# ---------------------------------------------------- reference fixtures
def _case(g, i):
    p = f"m{i}_"
    return int(g[p + "n"][0]), g[p + "row_ptr"], g[p + "col_idx"], g[p + "values"], g[p + "x"], p


def test_transforms_bit_exact_vs_reference(gpu, golden):
    sp = gpu
    for i in range(int(golden["count"][0])):
        n, rp, ci, v, x, p = _case(golden, i)
        m = upload(sp, n, rp, ci, v)
        ccs = m.convert(sp.Format.CCS)
        np.testing.assert_array_equal(ref_layout(ccs, sp, sp.Array.POINTER), golden[p + "ccs_col_ptr"])
        np.testing.assert_array_equal(ref_layout(ccs, sp, sp.Array.ROW_IDX), golden[p + "ccs_row_idx"])
        assert ccs.array(sp.Array.VALUES).tobytes() == golden[p + "ccs_values"].tobytes()
        for name, fmt in (("coo_row", sp.Format.COO_ROW), ("coo_col", sp.Format.COO_COL)):
            coo = m.convert(fmt)
            np.testing.assert_array_equal(ref_layout(coo, sp, sp.Array.ROW_IDX),
                                          golden[p + name + "_row_idx"])
            np.testing.assert_array_equal(ref_layout(coo, sp, sp.Array.COL_IDX),
                                          golden[p + name + "_col_idx"])
            assert coo.array(sp.Array.VALUES).tobytes() == golden[p + name + "_values"].tobytes()
        ell = m.convert(sp.Format.ELL)
        bc = int(golden[p + "ell_band_count"][0])
        assert ell.describe().band_count == bc
        assert ell.array(sp.Array.VALUES).tobytes() == golden[p + "ell_values"].tobytes()
        np.testing.assert_array_equal(ref_layout(ell, sp, sp.Array.COL_IDX), golden[p + "ell_col_idx"])
        np.testing.assert_array_equal(ell.array(sp.Array.ROW_ENTRY_COUNT, 8, 0),
                                      golden[p + "ell_row_entry_count"])
        # row-major ELL = transpose of the reference's band-major arrays
        rm = m.convert(sp.Format.ELL_ROWMAJOR)
        want_v = golden[p + "ell_values"].reshape(bc, n).T.reshape(-1) if bc else np.zeros(0)
        want_c = golden[p + "ell_col_idx"].reshape(bc, n).T.reshape(-1) if bc else np.zeros(0)
        assert rm.array(sp.Array.VALUES).tobytes() == np.ascontiguousarray(want_v).tobytes()
        np.testing.assert_array_equal(ref_layout(rm, sp, sp.Array.COL_IDX), want_c)


def test_spmv_all_kernels_vs_reference(gpu, golden):
    sp = gpu
    for i in range(int(golden["count"][0])):
        n, rp, ci, v, x, p = _case(golden, i)
        m = upload(sp, n, rp, ci, v)
        dense = dense_matvec(n, rp, ci, v, x)
        want = golden[p + "y_k0_l1"]
        y, t = m.spmv(x, sp.Kernel.CRS)
        assert max_rel_error(y, want) <= TOL and max_rel_error(y, dense) <= 1e-10
        for k, fmt in ((sp.Kernel.COO_ROW_OUTER, sp.Format.COO_ROW),
                       (sp.Kernel.COO_COL_OUTER, sp.Format.COO_COL),
                       (sp.Kernel.ELL_INNER, sp.Format.ELL),
                       (sp.Kernel.ELL_OUTER, sp.Format.ELL),
                       (sp.Kernel.ELL_ROWMAJOR, sp.Format.ELL_ROWMAJOR)):
            conv = m.convert(fmt)
            for lanes in (1, 3):
                y, _ = conv.spmv(x, k, lanes=lanes)
                ref_y = golden[p + f"y_k{min(int(k), 4) if k != sp.Kernel.ELL_ROWMAJOR else 3}_l{lanes}"]
                assert max_rel_error(y, ref_y) <= TOL, (i, k)
                assert max_rel_error(y, dense) <= 1e-10


def test_spmv_deterministic_where_reference_is(gpu):
    """Repeated calls are bitwise identical for every kernel except the
    column-ordered COO, whose fp64 reductions may add in any order (it stays
    within the 1e-12 contract; spmv.cpp:105-109 is lane-dependent too)."""
    sp = gpu
    rng = np.random.default_rng(37)
    for _ in range(5):
        n, rp, ci, v = random_crs(rng, 500, 20000)
        x = rng.uniform(-1, 1, n)
        m = upload(sp, n, rp, ci, v)
        for k, fmt in ((sp.Kernel.CRS, sp.Format.CRS), (sp.Kernel.COO_ROW_OUTER, sp.Format.COO_ROW),
                       (sp.Kernel.ELL_INNER, sp.Format.ELL), (sp.Kernel.ELL_OUTER, sp.Format.ELL),
                       (sp.Kernel.ELL_ROWMAJOR, sp.Format.ELL_ROWMAJOR)):
            h = m if fmt == sp.Format.CRS else m.convert(fmt)
            a, _ = h.spmv(x, k)
            b, _ = h.spmv(x, k)
            assert a.tobytes() == b.tobytes()


def test_padding_neutrality(gpu):
    """ELL padding slots (+0.0, own row) change nothing (test_spmv.cpp:172-190):
    a matrix with one long row forces padding in every other row."""
    sp = gpu
    rng = np.random.default_rng(41)
    n, rp, ci, v = random_crs(rng, 300, 3000)
    x = rng.uniform(-1, 1, n)
    m = upload(sp, n, rp, ci, v)
    want, _ = m.spmv(x, sp.Kernel.CRS)
    y, _ = m.convert(sp.Format.ELL).spmv(x, sp.Kernel.ELL_INNER)
    assert max_rel_error(y, want) <= TOL


def test_generators_byte_identical_to_reference(gpu, golden):
    sp = gpu
    gens = {
        "banded_200_1": lambda: sp.Matrix.gen_banded(200, 1),
        "banded_300_4": lambda: sp.Matrix.gen_banded(300, 4),
        "skewed_500_2_10_250_99": lambda: sp.Matrix.gen_skewed(500, 2, 10, 250, 99),
        "skewed_10000_1_1_5000_0": lambda: sp.Matrix.gen_skewed(10000, 1, 1, 5000, 0),
        "cv_2000_8_1.5_7": lambda: sp.Matrix.gen_cv_target(2000, 8.0, 1.5, 7),
        "cv_1000_5_0_3": lambda: sp.Matrix.gen_cv_target(1000, 5.0, 0.0, 3),
    }
    for key, make in gens.items():
        m = make()
        np.testing.assert_array_equal(ref_layout(m, sp, sp.Array.POINTER),
                                      golden[f"gen_{key}_row_ptr"])
        np.testing.assert_array_equal(ref_layout(m, sp, sp.Array.COL_IDX),
                                      golden[f"gen_{key}_col_idx"])
        assert m.array(sp.Array.VALUES).tobytes() == golden[f"gen_{key}_values"].tobytes()
    with pytest.raises(sp.SpmvtkError) as e:
        sp.Matrix.gen_banded(5, 5)
    assert e.value.status == sp.Status.ERR_USAGE
    with pytest.raises(sp.SpmvtkError) as e:
        sp.Matrix.gen_cv_target(100, 90.0, 3.0, 1)
    assert "feasible" in e.value.message


def test_larger_random_parity_with_port(gpu, port):
    """Bigger than the fixtures (long rows, many empty rows, unsorted columns)
    against the C port, bit-exact transforms + 1e-12 SpMV."""
    sp = gpu
    rng = np.random.default_rng(7)
    for it in range(4):
        n = int(rng.integers(2000, 6000))
        lens = rng.integers(0, 40, size=n)
        lens[rng.integers(0, n, size=3)] = rng.integers(3000, 6000, size=3)  # long rows
        lens[rng.random(n) < 0.2] = 0  # empty rows
        rows = [np.sort(rng.choice(n, size=min(int(l), n), replace=False)) for l in lens]
        for r in rows:
            rng.shuffle(r)
        ci = np.concatenate(rows).astype(np.int64) + 1
        rp = np.concatenate([[1], 1 + np.cumsum([len(r) for r in rows])]).astype(np.int64)
        v = rng.standard_normal(ci.shape[0])
        x = rng.uniform(-1, 1, n)
        m = upload(sp, n, rp, ci, v)
        cp, ri, cv = port.crs_to_ccs(n, rp, ci, v)
        ccs = m.convert(sp.Format.CCS)
        np.testing.assert_array_equal(ref_layout(ccs, sp, sp.Array.POINTER), cp)
        np.testing.assert_array_equal(ref_layout(ccs, sp, sp.Array.ROW_IDX), ri)
        assert ccs.array(sp.Array.VALUES).tobytes() == cv.tobytes()
        bc, ev, ec, cnt = port.crs_to_ell(n, rp, ci, v)
        ell = m.convert(sp.Format.ELL)
        assert ell.array(sp.Array.VALUES).tobytes() == ev.tobytes()
        np.testing.assert_array_equal(ref_layout(ell, sp, sp.Array.COL_IDX), ec)
        want = port.spmv_crs(n, rp, ci, v, x)
        for k, f in ((sp.Kernel.CRS, None), (sp.Kernel.COO_ROW_OUTER, sp.Format.COO_ROW),
                     (sp.Kernel.COO_COL_OUTER, sp.Format.COO_COL), (sp.Kernel.ELL_INNER, sp.Format.ELL),
                     (sp.Kernel.ELL_OUTER, sp.Format.ELL),
                     (sp.Kernel.ELL_ROWMAJOR, sp.Format.ELL_ROWMAJOR)):
            h = m if f is None else m.convert(f)
            y, _ = h.spmv(x, k)
            assert max_rel_error(y, want) <= TOL, (it, k)


def _crs_from_pairs(n, r, c, rng):
    key = np.unique(r.astype(np.int64) * n + c.astype(np.int64))
    rows, cols = key // n, key % n
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]).astype(np.int64) + 1
    return rp, cols.astype(np.int64) + 1, rng.standard_normal(key.shape[0])


def test_ccs_partition_paths(gpu, port):
    """CRS->CCS through each partition path against the C port, bit-exact:
    scattered columns (many runs -> coarse pass + refine) with a 1000-entry
    column (block network inside a bucket) and two dense columns (oversized
    bucket path); a banded matrix (few runs -> single pass); a matrix whose
    slices split between the windowed staged scatter and the cursor scatter.
    Both with and without the windowed staged pass."""
    sp = gpu
    rng = np.random.default_rng(21)
    n = 300_000
    r = np.repeat(np.arange(n), rng.integers(4, 20, size=n))
    c = rng.integers(0, n, size=r.shape[0])
    dense = rng.random(n) < 0.5
    extra_r = np.concatenate([np.nonzero(dense)[0], np.nonzero(dense)[0],
                              rng.choice(n, 1000, replace=False)])
    extra_c = np.concatenate([np.full(dense.sum(), 5), np.full(dense.sum(), 77777),
                              np.full(1000, 123456)])
    cases = [(n, *_crs_from_pairs(n, np.concatenate([r, extra_r]),
                                  np.concatenate([c, extra_c]), rng))]
    nb = 200_000
    rb = np.repeat(np.arange(nb), 24)
    cb = np.clip(rb + rng.integers(-500, 500, size=rb.shape[0]), 0, nb - 1)
    cases.append((nb, *_crs_from_pairs(nb, rb, cb, rng)))
    # mixed single pass: banded slices (narrow bucket windows -> staged) and,
    # in the last eighth of the rows, scattered slices (every bucket -> cursor
    # scatter), with few enough runs to stay single-pass
    nm = 1 << 20
    rm = np.repeat(np.arange(nm), 8)
    cm = np.clip(rm + rng.integers(-2000, 2000, size=rm.shape[0]), 0, nm - 1)
    tail = rm >= nm - nm // 8
    cm[tail] = rng.integers(0, nm, size=int(tail.sum()))
    cases.append((nm, *_crs_from_pairs(nm, rm, cm, rng)))
    lib = sp.load_library()
    try:
        for window in (1, 0):
            lib.spmvtk_k_tune(b"ccs_window", window)
            for nn, rp, ci, v in cases:
                m = upload(sp, nn, rp, ci, v)
                cp, ri, cv = port.crs_to_ccs(nn, rp, ci, v)
                ccs = m.convert(sp.Format.CCS)
                np.testing.assert_array_equal(ref_layout(ccs, sp, sp.Array.POINTER), cp)
                np.testing.assert_array_equal(ref_layout(ccs, sp, sp.Array.ROW_IDX), ri)
                assert ccs.array(sp.Array.VALUES).tobytes() == cv.tobytes()
                ccs.free()
                m.free()
    finally:
        lib.spmvtk_k_tune(b"ccs_window", 1)


def test_crs_long_rows_path(gpu, port):
    """Rows above the vector kernel's 4096 limit take the block-per-row pass."""
    sp = gpu
    rng = np.random.default_rng(11)
    n = 20000
    lens = rng.integers(0, 8, size=n)
    lens[[5, 77, 19999]] = [20000, 9000, 4097]
    rows = [np.sort(rng.choice(n, size=int(l), replace=False)) for l in lens]
    ci = np.concatenate(rows).astype(np.int64) + 1
    rp = np.concatenate([[1], 1 + np.cumsum(lens)]).astype(np.int64)
    v = rng.standard_normal(ci.shape[0])
    x = rng.uniform(-1, 1, n)
    m = upload(sp, n, rp, ci, v)
    y, _ = m.spmv(x, sp.Kernel.CRS)
    assert max_rel_error(y, port.spmv_crs(n, rp, ci, v, x)) <= TOL


# -------------------------------------------- the reference's C API scenario
def test_capi_end_to_end(gpu, kat):
    """Mirror of test_capi.cpp:29-141 through our C ABI."""
    sp = gpu
    c = kat["capi_banded"]
    banded = sp.Matrix.gen_banded(c["n"], c["half_width"])
    info = banded.info()
    assert info.n == c["n"] and info.nnz == c["nnz"] and info.max_row_entries == c["max_row_entries"]
    assert info.d_mat > 0
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "banded.mtx")
        banded.write_matrix_market(path)
        back = sp.Matrix.read_matrix_market(path)
        info2 = back.info()
        assert info2.nnz == info.nnz and info2.d_mat == info.d_mat
        x = np.ones(c["n"])
        y0, _ = banded.spmv(x, sp.Kernel.CRS)
        for fmt, k in ((sp.Format.COO_ROW, sp.Kernel.COO_ROW_OUTER),
                       (sp.Format.COO_COL, sp.Kernel.COO_COL_OUTER),
                       (sp.Format.ELL, sp.Kernel.ELL_INNER), (sp.Format.ELL, sp.Kernel.ELL_OUTER)):
            conv = banded.convert(fmt)
            assert conv.format == fmt
            y, _ = conv.spmv(x, k, lanes=3)
            assert np.all(np.abs(y - y0) <= 1e-12 * np.abs(y0))
            # non-CRS handles are written through their CRS reconstruction
            p2 = os.path.join(d, f"conv{int(fmt)}.mtx")
            conv.write_matrix_market(p2)
            assert open(p2).read() == open(path).read()
        b = sp.bench(banded, sp.Kernel.ELL_OUTER, 1, 3, 0)
        assert b["t_crs"] > 0 and b["sp"] > 0 and b["t_trans"] > 0
        assert b["r"] == pytest.approx(b["sp"] / b["tt"])
        second = sp.Matrix.gen_banded(200, 2)
        prof = sp.Profile.build([banded, second], ["a", "b"], sp.Kernel.ELL_INNER, 1, 1.0, 3, 0,
                                "capi-test")
        recs = prof.records()
        assert len(recs) == 2 and recs[0]["matrix_id"] == "a"
        assert not recs[0]["excluded"] and recs[0]["r"] > 0
        ppath = os.path.join(d, "profile.json")
        prof.write(ppath)
        back_p = sp.Profile.read(ppath)
        assert back_p.d_star == prof.d_star and back_p.kernel == sp.Kernel.ELL_INNER
        dec, dm = sp.select(banded, back_p)
        assert dm > 0
        bad = os.path.join(d, "bad.json")
        open(bad, "w").write('{"version": 1, "oops": true}')
        with pytest.raises(sp.SpmvtkError) as e:
            sp.Profile.read(bad)
        assert e.value.status == sp.Status.ERR_DATA
    assert sp.last_error() != ""


def test_online_select_strict(gpu, kat, ref):
    sp = gpu
    c = kat["online_select"]
    banded = sp.Matrix.gen_banded(*c["banded"])
    skew = sp.Matrix.gen_skewed(*c["skewed"])
    # profile with d_star = 0.1 through the JSON reader (schema v1)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "p.json")
        open(path, "w").write('{"version": 1, "machine_label": "x", "kernel_variant": '
                              '"ell-inner", "lanes": 1, "c": 1.0, "d_star": 0.1, "records": []}')
        p = sp.Profile.read(path)
        dec, dm = sp.select(banded, p)
        assert dec == sp.Decision.USE_ELL
        dec2, dm2 = sp.select(skew, p)
        assert dm2 > 0.1 and dec2 == sp.Decision.USE_CRS
        open(path, "w").write('{"version": 1, "machine_label": "x", "kernel_variant": '
                              '"ell-inner", "lanes": 1, "c": 1.0, "d_star": %r, "records": []}' % dm)
        p2 = sp.Profile.read(path)
        assert sp.select(banded, p2)[0] == sp.Decision.USE_CRS  # strict
    # GPU D_mat vs the reference Welford value
    hb = ref.gen("banded", *c["banded"])
    assert dm == pytest.approx(ref.row_stats(hb)[2], rel=1e-12)
    ref.free(hb)


def test_profile_excludes_guarded_matrix(gpu):
    sp = gpu
    ok = sp.Matrix.gen_banded(300, 1)
    n = 10000
    rp = np.full(n + 1, 5001, np.int64)
    rp[0] = 1
    wide = upload(sp, n, rp, np.arange(1, 5001), np.ones(5000))
    p = sp.Profile.build([ok, wide], ["ok", "overflow"], sp.Kernel.ELL_OUTER, 1, 1.0, 3,
                         100 << 20)
    recs = p.records()
    assert not recs[0]["excluded"] and recs[1]["excluded"]
    assert "exceeds" in recs[1]["exclusion_reason"]
    assert np.isnan(recs[1]["r"])
    with pytest.raises(sp.SpmvtkError) as e:
        sp.Profile.build([ok], ["ok"], sp.Kernel.CRS)
    assert e.value.status == sp.Status.ERR_USAGE


def test_validation_rejects_bad_arrays(gpu):
    sp = gpu
    with pytest.raises(sp.SpmvtkError) as e:
        sp.Matrix.from_crs(2, np.array([0, 2, 1]), np.array([0, 1]), np.ones(2))
    assert e.value.status == sp.Status.ERR_DATA
    with pytest.raises(sp.SpmvtkError):
        sp.Matrix.from_crs(2, np.array([0, 1, 2]), np.array([0, 5]), np.ones(2))
    with pytest.raises(sp.SpmvtkError) as e:
        sp.Matrix.from_crs(2, np.array([1, 1, 2]), np.array([0]), np.ones(1), index_base=0)
    assert e.value.status == sp.Status.ERR_DATA


def test_coo_row_kernels_both_variants(gpu, port):
    """The 4-entries-per-lane COO-row kernel (default) and the scalar one agree
    with the oracle on matrices with empty rows, long rows spanning many warp
    chunks and row runs crossing lane / group boundaries."""
    sp = gpu
    lib = sp.load_library()
    rng = np.random.default_rng(99)
    try:
        for it in range(6):
            n = int(rng.integers(1, 5000))
            lens = rng.integers(0, 12, size=n)
            lens[rng.random(n) < 0.3] = 0
            if it % 2:
                lens[rng.integers(0, n, size=2)] = rng.integers(2000, 9000, size=2)
            lens = np.minimum(lens, n)
            rows = [np.sort(rng.choice(n, size=int(l), replace=False)) for l in lens]
            ci = (np.concatenate(rows) if rows else np.zeros(0)).astype(np.int64) + 1
            rp = np.concatenate([[1], 1 + np.cumsum(lens)]).astype(np.int64)
            v = rng.standard_normal(ci.shape[0])
            x = rng.uniform(-1, 1, n)
            want = port.spmv_crs(n, rp, ci, v, x)
            coo = upload(sp, n, rp, ci, v).convert(sp.Format.COO_ROW)
            ys = []
            for variant in (1, 0):
                lib.spmvtk_k_tune(b"coo_variant", variant)
                y, _ = coo.spmv(x, sp.Kernel.COO_ROW_OUTER)
                assert max_rel_error(y, want) <= TOL, (it, variant)
                ys.append(y)
    finally:
        lib.spmvtk_k_tune(b"coo_variant", 1)


def test_pipelined_host_spmv_matches_device(gpu):
    """spmvtk_spmv with pinned host buffers takes the row-chunked pipeline
    (D2H of finished rows overlaps the SpMV of the next); results must be
    bitwise those of the pageable (single-shot) call and the device call."""
    import torch
    sp = gpu
    m = sp.HostCrs(2, 1 << 16).upload()
    n = m.describe().n
    x = sp.gen_vector(n, 5)
    xp = torch.from_numpy(x.copy()).pin_memory()
    for h, k in ((m, sp.Kernel.CRS), (m.convert(sp.Format.ELL), sp.Kernel.ELL_INNER),
                 (m.convert(sp.Format.ELL_ROWMAJOR), sp.Kernel.ELL_ROWMAJOR)):
        yp = torch.empty(n, dtype=torch.float64).pin_memory()
        h.spmv(xp.numpy(), k, 1, out=yp.numpy())
        y_pageable, _ = h.spmv(x, k)
        assert yp.numpy().tobytes() == y_pageable.tobytes(), k


def test_streaming_pipeline_matches_spmv(gpu):
    """spmvtk_pipeline_*: several products in flight (double-buffered device
    staging, copy-in / SpMV / copy-out on three streams) give bitwise the
    results of the synchronous spmvtk_spmv for every submitted x."""
    import torch
    sp = gpu
    m = sp.HostCrs(2, 1 << 15).upload()
    n = m.describe().n
    for h, k in ((m, sp.Kernel.CRS), (m.convert(sp.Format.ELL), sp.Kernel.ELL_INNER),
                 (m.convert(sp.Format.COO_ROW), sp.Kernel.COO_ROW_OUTER)):
        pipe = sp.Pipeline(h, k)
        xs = [torch.from_numpy(sp.gen_vector(n, 100 + i)).pin_memory() for i in range(5)]
        ys = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(5)]
        for x, y in zip(xs, ys):
            pipe.submit(x.numpy(), y.numpy())
        pipe.wait()
        for x, y in zip(xs, ys):
            want, _ = h.spmv(x.numpy(), k)
            assert y.numpy().tobytes() == want.tobytes(), k
        pipe.free()


def test_concurrent_threads_share_a_handle(gpu):
    """Handles are immutable and safe for concurrent reads (SPEC.md:100-101,
    SURVEY.md 8b): 4 host threads, each on its own CUDA stream, run SpMVs,
    conversions and statistics on one handle at once; every result equals
    the single-threaded one bitwise."""
    import threading

    import torch
    sp = gpu
    m = sp.HostCrs(2, 1 << 16).upload()
    n = m.describe().n
    xs = [sp.gen_vector(n, 50 + i) for i in range(4)]
    want = [m.spmv(x, sp.Kernel.CRS)[0] for x in xs]
    ell_want = m.convert(sp.Format.ELL)
    want_ell = [ell_want.spmv(x, sp.Kernel.ELL_INNER)[0] for x in xs]
    errors = []

    def work(i):
        try:
            stream = torch.cuda.Stream()
            sp.set_stream(stream.cuda_stream)  # thread-local
            for _ in range(5):
                y, _ = m.spmv(xs[i], sp.Kernel.CRS)
                assert y.tobytes() == want[i].tobytes()
                e = m.convert(sp.Format.ELL)
                y2, _ = e.spmv(xs[i], sp.Kernel.ELL_INNER)
                assert y2.tobytes() == want_ell[i].tobytes()
                e.free()
                assert m.row_stats().max_row == m.info().max_row_entries
        except Exception as ex:  # noqa: BLE001
            errors.append(f"thread {i}: {ex!r}")

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_row_block_shards_single_gpu(gpu, port):
    """Row-block shards (the multi-GPU layout) run on one GPU: per-shard
    SpMV assembled == full SpMV (1e-12), and each shard's ELL equals the
    reference ELL of its row block embedded in the n x n matrix (padding
    column = global row index)."""
    from paper_2407_00019_b200 import dist as D
    sp = gpu
    rng = np.random.default_rng(5)
    n, rp, ci, v = random_crs(rng, 3000, 60000)
    x = rng.uniform(-1, 1, n)
    want = port.spmv_crs(n, rp, ci, v, x)
    rp0, ci0 = rp - 1, ci - 1
    kernels = ((sp.Kernel.CRS, None), (sp.Kernel.ELL_INNER, sp.Format.ELL),
               (sp.Kernel.COO_ROW_OUTER, sp.Format.COO_ROW),
               (sp.Kernel.ELL_ROWMAJOR, sp.Format.ELL_ROWMAJOR))
    for world in (2, 3, 4):
        parts = {k: [] for k, _ in kernels}
        for r in range(world):
            r0, lrp, lci, lv = D.shard_arrays(rp0, ci0, v, n, world, r)
            rows = D.block_rows(n, world)
            sh = sp.Matrix.from_crs_block(rows, n, r0, lrp, lci, lv)
            d = sh.describe()
            assert (d.n, d.ncols, d.row_offset) == (rows, n, r0)
            for k, f in kernels:
                h = sh if f is None else sh.convert(f)
                y, _ = h.spmv(x, k)
                assert y.shape[0] == rows
                parts[k].append(y[: D.block_range(n, world, r)[1] - r0])
            # ELL arrays of the shard vs the reference ELL of the embedded block
            a, b = D.block_range(n, world, r)
            erp = np.concatenate([np.full(a, rp[a]), rp[a:b + 1],
                                  np.full(n - b, rp[b])]).astype(np.int64)
            erp = erp - erp[0] + 1
            sl = slice(rp[a] - 1, rp[b] - 1)
            bc, ev, ec, cnt = port.crs_to_ell(n, erp, ci[sl], v[sl])
            ell = sh.convert(sp.Format.ELL)
            assert ell.describe().band_count == bc
            got_v = ell.array(sp.Array.VALUES).reshape(bc, rows) if bc else np.zeros((0, rows))
            got_c = ell.array(sp.Array.COL_IDX, 8, 1).reshape(bc, rows) if bc else None
            want_v = ev.reshape(bc, n)[:, a:b] if bc else np.zeros((0, b - a))
            assert got_v[:, : b - a].tobytes() == np.ascontiguousarray(want_v).tobytes()
            if bc:
                np.testing.assert_array_equal(got_c[:, : b - a], ec.reshape(bc, n)[:, a:b])
        for k, _ in kernels:
            assert max_rel_error(np.concatenate(parts[k]), want) <= TOL, (world, k)
    with pytest.raises(sp.SpmvtkError) as e:
        sp.Matrix.from_crs_block(2, 10, 0, np.array([0, 1, 2]), np.array([3, 9]),
                                 np.ones(2)).convert(sp.Format.CCS)
    assert e.value.status == sp.Status.ERR_USAGE


def test_inverse_conversions_on_device(gpu, golden):
    """coo_to_crs / ell_to_crs / CCS->CRS / canonicalize on the GPU give the
    canonical CRS (test_convert.cpp:146-177, acceptance.cpp:90-115)."""
    sp = gpu
    for i in range(int(golden["count"][0])):
        n, rp, ci, v, x, p = _case(golden, i)
        m = upload(sp, n, rp, ci, v)
        # canonical reference: sort columns inside each row
        crp = np.asarray(rp, np.int64)
        order = np.concatenate([np.argsort(ci[crp[r] - 1:crp[r + 1] - 1], kind="stable") +
                                crp[r] - 1 for r in range(n)]).astype(np.int64) \
            if v.size else np.zeros(0, np.int64)
        want_c, want_v = ci[order], v[order]
        for h in (m, m.convert(sp.Format.CCS), m.convert(sp.Format.COO_ROW),
                  m.convert(sp.Format.COO_COL), m.convert(sp.Format.ELL),
                  m.convert(sp.Format.ELL_ROWMAJOR)):
            c = h.to_crs()
            assert c.format == sp.Format.CRS
            np.testing.assert_array_equal(c.array(sp.Array.POINTER), crp)
            np.testing.assert_array_equal(c.array(sp.Array.COL_IDX), want_c)
            assert c.array(sp.Array.VALUES).tobytes() == want_v.tobytes()
    # duplicates are refused with the reference message
    dup = sp.Matrix.from_crs(2, np.array([0, 2, 3]), np.array([1, 1, 0]), np.ones(3))
    coo = dup.convert(sp.Format.COO_ROW)
    with pytest.raises(sp.SpmvtkError) as e:
        coo.to_crs()
    assert e.value.status == sp.Status.ERR_DATA and "duplicate (row, col) pair (1, 2)" in \
        e.value.message


def test_lower_abi_phase1_phase2_and_statistics(gpu, port):
    """The lower C ABI (spmvtk_kernels.h) called directly on device buffers:
    spmvtk_k_crs_to_coo_col (Phase I with Phase II fused), spmvtk_k_expand_ptr
    (Phase II alone, on the col_ptr of spmvtk_k_crs_to_ccs) and
    spmvtk_k_row_stats_mapped (max/sum/sumsq published into mapped memory,
    accumulator left zeroed for the next call) -- against the C port."""
    import ctypes as C

    import torch
    sp = gpu
    lib = sp.load_library()
    P, I64, U64 = C.c_void_p, C.c_int64, C.c_uint64
    lib.spmvtk_k_ccs_scratch_bytes.restype = C.c_size_t
    lib.spmvtk_k_ccs_scratch_bytes.argtypes = [I64, I64]
    lib.spmvtk_k_crs_to_ccs.argtypes = [I64, I64, P, P, P, P, P, P, P, P]
    lib.spmvtk_k_crs_to_coo_col.argtypes = [I64, I64, P, P, P, P, P, P, P, P, P]
    lib.spmvtk_k_expand_ptr.argtypes = [P, I64, I64, P, P]
    lib.spmvtk_k_row_stats_mapped.argtypes = [P, I64, P, P, U64, P]
    rng = np.random.default_rng(5)
    n = 40_000
    lens = rng.integers(0, 30, size=n)
    rows = [np.sort(rng.choice(n, size=int(ln), replace=False)) for ln in lens]
    ci = np.concatenate(rows)
    rp = np.concatenate([[0], np.cumsum(lens)])
    v = rng.standard_normal(ci.shape[0])
    nnz = int(rp[-1])
    dev = lambda a, dt: torch.as_tensor(np.asarray(a, dt), device="cuda")  # noqa: E731
    irp, icol, val = dev(rp, np.int32), dev(ci, np.int32), dev(v, np.float64)
    stream = torch.cuda.current_stream().cuda_stream
    scratch = torch.empty(lib.spmvtk_k_ccs_scratch_bytes(n, nnz), dtype=torch.uint8, device="cuda")
    cp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    ri = torch.empty(nnz, dtype=torch.int32, device="cuda")
    cc = torch.empty(nnz, dtype=torch.int32, device="cuda")
    cv = torch.empty(nnz, dtype=torch.float64, device="cuda")
    assert lib.spmvtk_k_crs_to_coo_col(n, nnz, irp.data_ptr(), icol.data_ptr(), val.data_ptr(),
                                       cp.data_ptr(), ri.data_ptr(), cc.data_ptr(),
                                       cv.data_ptr(), scratch.data_ptr(), stream) == 0
    want_r, want_c, want_v = port.crs_to_coo_col(n, rp + 1, ci + 1, v)
    np.testing.assert_array_equal(ri.cpu().numpy() + 1, want_r)
    np.testing.assert_array_equal(cc.cpu().numpy() + 1, want_c)
    assert cv.cpu().numpy().tobytes() == want_v.tobytes()
    # Phase I alone, then Phase II from its col_ptr
    ri2 = torch.empty_like(ri)
    cv2 = torch.empty_like(cv)
    assert lib.spmvtk_k_crs_to_ccs(n, nnz, irp.data_ptr(), icol.data_ptr(), val.data_ptr(),
                                   cp.data_ptr(), ri2.data_ptr(), cv2.data_ptr(),
                                   scratch.data_ptr(), stream) == 0
    cc2 = torch.empty_like(cc)
    assert lib.spmvtk_k_expand_ptr(cp.data_ptr(), n, nnz, cc2.data_ptr(), stream) == 0
    assert torch.equal(ri2, ri) and torch.equal(cc2, cc) and torch.equal(cv2, cv)
    # column indices starting 4/8/12 bytes past a 16-byte boundary (the
    # bucket count reads them with 16-byte loads over the aligned body)
    for shift in (1, 2, 3):
        buf = torch.empty(nnz + 4, dtype=torch.int32, device="cuda")
        icol_u = buf[shift:shift + nnz]
        icol_u.copy_(icol)
        ri3, cv3 = torch.empty_like(ri), torch.empty_like(cv)
        assert lib.spmvtk_k_crs_to_ccs(n, nnz, irp.data_ptr(), icol_u.data_ptr(), val.data_ptr(),
                                       cp.data_ptr(), ri3.data_ptr(), cv3.data_ptr(),
                                       scratch.data_ptr(), stream) == 0
        assert torch.equal(ri3, ri) and torch.equal(cv3, cv), shift
    # row statistics through mapped memory, twice (the accumulator resets)
    acc = torch.zeros(4, dtype=torch.int64, device="cuda")
    host = torch.zeros(4, dtype=torch.int64).pin_memory()
    for seq in (1, 2):
        assert lib.spmvtk_k_row_stats_mapped(irp.data_ptr(), n, acc.data_ptr(), host.data_ptr(),
                                             seq, stream) == 0
        torch.cuda.synchronize()
        h = host.numpy()
        assert int(h[3]) == seq
        assert int(h[0]) == int(lens.max())
        assert int(h[1]) == int(lens.sum())
        assert int(h[2]) == int((lens.astype(np.int64) ** 2).sum())
        assert int(acc.abs().sum().item()) == 0


def test_lower_abi_spmv_kernels_on_unaligned_arrays(gpu, port):
    """spmvtk_k_spmv_crs_seg and spmvtk_k_spmv_coo_row on device arrays that
    start 4 / 8 bytes past an aligned address (arrays a caller hands in
    through the lower ABI need not be pool-aligned): the 256-bit / 128-bit
    loads must switch off, the products stay within 1e-12 of the port."""
    import ctypes as C

    import torch
    sp = gpu
    lib = sp.load_library()
    P, I64, I32 = C.c_void_p, C.c_int64, C.c_int32
    lib.spmvtk_k_seg_plan_warps.restype = C.c_int32
    lib.spmvtk_k_seg_plan_warps.argtypes = [I64, I32]
    lib.spmvtk_k_seg_plan.argtypes = [I64, I64, P, I32, P, P]
    lib.spmvtk_k_spmv_crs_seg.argtypes = [P, P, P, P, P, P, I32, I32, I64, I64, I64, P]
    lib.spmvtk_k_spmv_coo_row.argtypes = [I64, I64, P, P, P, P, P, P]
    rng = np.random.default_rng(17)
    n = 30_000
    lens = np.minimum(n, np.round(rng.lognormal(2.0, 1.2, size=n)).astype(np.int64))
    rows = [np.sort(rng.choice(n, size=int(ln), replace=False)) for ln in lens]
    ci = np.concatenate(rows).astype(np.int32)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    v = rng.standard_normal(ci.shape[0])
    nnz = int(rp[-1])
    x = rng.uniform(-1, 1, n)
    want = port.spmv_crs(n, rp.astype(np.int64) + 1, ci.astype(np.int64) + 1, v, x)  # 1-based
    stream = torch.cuda.current_stream().cuda_stream

    def shifted(a, dt, shift_elems):
        buf = torch.empty(a.shape[0] + 8, dtype=dt, device="cuda")
        view = buf[shift_elems:shift_elems + a.shape[0]]
        view.copy_(torch.from_numpy(a))
        return view

    irp = torch.from_numpy(rp).cuda()
    xd = torch.from_numpy(x).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    chunk = 2048
    nw = lib.spmvtk_k_seg_plan_warps(nnz, chunk)
    plan = torch.empty(nw + 1, dtype=torch.int32, device="cuda")
    assert lib.spmvtk_k_seg_plan(n, nnz, irp.data_ptr(), chunk, plan.data_ptr(), stream) == 0
    rows_coo = np.repeat(np.arange(n, dtype=np.int32), lens)
    for cshift, vshift in ((0, 0), (1, 1), (0, 1), (2, 3)):
        icol = shifted(ci, torch.int32, cshift)
        val = shifted(v, torch.float64, vshift)
        y.fill_(float("nan"))
        assert lib.spmvtk_k_spmv_crs_seg(irp.data_ptr(), icol.data_ptr(), val.data_ptr(),
                                         xd.data_ptr(), y.data_ptr(), plan.data_ptr(), 0, nw, 0,
                                         n, nnz, stream) == 0
        assert np.max(np.abs(y.cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(want)), (cshift, vshift)
        rowd = shifted(rows_coo, torch.int32, cshift)
        y.fill_(float("nan"))
        assert lib.spmvtk_k_spmv_coo_row(n, nnz, rowd.data_ptr(), icol.data_ptr(), val.data_ptr(),
                                         xd.data_ptr(), y.data_ptr(), stream) == 0
        assert np.max(np.abs(y.cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(want)), (cshift, vshift)
