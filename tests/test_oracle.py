"""Pins the oracle before anything is checked against it (CPU only).

1. The plain-C restatement (oracle/spmvtk_oracle.c) reproduces every
   known-answer vector restated from the reference's own tests
   (tests/golden/kat.json, each entry cites test file:line).
2. It reproduces, bit for bit, the outputs of the reference library itself on
   seeded random matrices (tests/golden/ref_random.npz, produced by
   tests/golden/make_golden.py from /root/reference compiled as-is).
3. When oracle/_ref is present it is also checked live on fresh inputs.
"""
import os

import numpy as np
import pytest

from oracle.oracle import REF_LIB, Ref, dense_matvec, max_rel_error, random_crs


def test_kat_coo_row(port, kat):
    for c in kat["coo_row"]:
        r, col, v = port.crs_to_coo_row(c["n"], c["row_ptr"], c["col_idx"], c["values"])
        assert r.tolist() == c["row_idx"], c["ref"]
        assert col.tolist() == c["out_col_idx"], c["ref"]
        assert v.tolist() == c["out_values"], c["ref"]


def test_kat_ccs_and_coo_col(port, kat):
    for c in kat["ccs"]:
        cp, ri, v = port.crs_to_ccs(c["n"], c["row_ptr"], c["col_idx"], c["values"])
        assert cp.tolist() == c["col_ptr"], c["ref"]
        assert ri.tolist() == c["row_idx"], c["ref"]
        assert v.tolist() == c["out_values"], c["ref"]
    for c in kat["coo_col"]:
        r, col, v = port.crs_to_coo_col(c["n"], c["row_ptr"], c["col_idx"], c["values"])
        assert col.tolist() == c["out_col_idx"] and r.tolist() == c["row_idx"]
        assert v.tolist() == c["out_values"]


def test_kat_ell(port, kat):
    for c in kat["ell"]:
        bc, v, col, cnt = port.crs_to_ell(c["n"], c["row_ptr"], c["col_idx"], c["values"])
        assert bc == c["band_count"], c["ref"]
        assert int(cnt.sum()) == c["stored_nnz"]
        assert cnt.tolist() == c["row_entry_count"]
        if "out_values" in c:
            assert v.tolist() == c["out_values"]
            assert col.tolist() == c["out_col_idx"]
    g = kat["ell_guard"]
    n = g["n"]
    rp = np.full(n + 1, g["heavy_row_entries"] + 1, np.int64)
    rp[0] = 1
    ci = np.arange(1, g["heavy_row_entries"] + 1)
    with pytest.raises(MemoryError, match=g["message_contains"]):
        port.crs_to_ell(n, rp, ci, np.ones(ci.shape[0]), max_bytes=g["max_bytes"])


def test_kat_estimate_and_partition(port, kat):
    for c in kat["estimate_ell_bytes"]:
        assert port.estimate_ell_bytes(c["n"], c["row_ptr"], c["value_bytes"],
                                       c["index_bytes"]) == c["bytes"], c["ref"]
    for c in kat["partition_range"]:
        if c.get("error"):
            with pytest.raises(ValueError):
                port.partition_range(c["len"], c["lanes"])
        else:
            s, e = port.partition_range(c["len"], c["lanes"])
            assert s.tolist() == c["istart"] and e.tolist() == c["iend"], c["ref"]


def test_kat_spmv(port, kat):
    for c in kat["spmv_crs"]:
        y = port.spmv_crs(c["n"], c["row_ptr"], c["col_idx"], c["values"], c["x"])
        assert y.tolist() == c["y"], c["ref"]
    c = kat["ell_padding_spmv"]
    bc, v, col, _ = port.crs_to_ell(c["n"], c["row_ptr"], c["col_idx"], c["values"])
    assert port.spmv_ell_inner(c["n"], bc, v, col, c["x"]).tolist() == c["y"]
    assert port.spmv_ell_outer(c["n"], bc, v, col, c["x"], 2).tolist() == c["y"]
    c = kat["ell_outer_idle_lanes"]
    n = c["n"]
    bc, v, col, _ = port.crs_to_ell(n, np.arange(1, n + 2), np.arange(1, n + 1), np.ones(n))
    assert port.spmv_ell_outer(n, bc, v, col, c["x"], c["lanes"]).tolist() == c["y"]


def test_kat_stats(port, kat):
    for c in kat["stats"]:
        counts = np.array(c["counts"], np.int64)
        rp = np.concatenate([[1], 1 + np.cumsum(counts)])
        mu, sg, dm = port.row_stats(len(counts), rp)
        if c.get("exact"):
            assert dm == c["d_mat"], c["ref"]
            if "mu" in c:
                assert mu == c["mu"] and sg == c["sigma"]
        elif "d_mat" in c:
            assert mu == pytest.approx(c["mu"], rel=1e-15)
            assert sg == pytest.approx(c["sigma"], rel=1e-15)
            assert dm == pytest.approx(c["d_mat"], rel=1e-15)
        if c.get("d_mat_positive"):
            assert dm > 0
    with pytest.raises(ValueError):
        port.row_stats(3, [1, 1, 1, 1])


def test_kat_autotune_arithmetic(port, kat):
    for c in kat["compute_metrics"]:
        if c.get("error"):
            with pytest.raises(ValueError):
                port.compute_metrics(*c["t"])
        else:
            assert port.compute_metrics(*c["t"]) == (c["sp"], c["tt"], c["r"]), c["ref"]
    for c in kat["amortization"]:
        assert port.amortization(*c["t"]) == c["k"], c["ref"]
    for c in kat["find_d_star"]:
        assert port.find_d_star([tuple(r) for r in c["records"]], c["c"]) == c["d_star"], c["ref"]


def _golden_case(g, i):
    p = f"m{i}_"
    return (int(g[p + "n"][0]), g[p + "row_ptr"], g[p + "col_idx"], g[p + "values"], g[p + "x"], p)


def test_port_matches_reference_outputs_bitwise(port, golden):
    """Transforms bit-identical; sequential kernels bit-identical; lane-split
    kernels bit-identical too (same partition / reduction order)."""
    for i in range(int(golden["count"][0])):
        n, rp, ci, v, x, p = _golden_case(golden, i)
        cp, ri, cv = port.crs_to_ccs(n, rp, ci, v)
        np.testing.assert_array_equal(cp, golden[p + "ccs_col_ptr"])
        np.testing.assert_array_equal(ri, golden[p + "ccs_row_idx"])
        assert cv.tobytes() == golden[p + "ccs_values"].tobytes()
        for name, fn in (("coo_row", port.crs_to_coo_row), ("coo_col", port.crs_to_coo_col)):
            r, c, vv = fn(n, rp, ci, v)
            np.testing.assert_array_equal(r, golden[p + name + "_row_idx"])
            np.testing.assert_array_equal(c, golden[p + name + "_col_idx"])
            assert vv.tobytes() == golden[p + name + "_values"].tobytes()
        bc, ev, ec, cnt = port.crs_to_ell(n, rp, ci, v)
        assert bc == int(golden[p + "ell_band_count"][0])
        assert ev.tobytes() == golden[p + "ell_values"].tobytes()
        np.testing.assert_array_equal(ec, golden[p + "ell_col_idx"])
        np.testing.assert_array_equal(cnt, golden[p + "ell_row_entry_count"])
        y0 = port.spmv_crs(n, rp, ci, v, x)
        assert y0.tobytes() == golden[p + "y_k0_l1"].tobytes()
        rr, rc, rv = port.crs_to_coo_row(n, rp, ci, v)
        cr, cc, cv2 = port.crs_to_coo_col(n, rp, ci, v)
        for lanes in (1, 3):
            assert port.spmv_coo(n, rr, rc, rv, x, lanes).tobytes() == \
                golden[p + f"y_k1_l{lanes}"].tobytes()
            assert port.spmv_coo(n, cr, cc, cv2, x, lanes).tobytes() == \
                golden[p + f"y_k2_l{lanes}"].tobytes()
            assert port.spmv_ell_outer(n, bc, ev, ec, x, lanes).tobytes() == \
                golden[p + f"y_k4_l{lanes}"].tobytes()
            assert port.spmv_ell_inner(n, bc, ev, ec, x).tobytes() == \
                golden[p + f"y_k3_l{lanes}"].tobytes()


def test_port_against_dense_oracle():
    from oracle.oracle import Port
    port = Port()
    rng = np.random.default_rng(31)
    for _ in range(20):
        n, rp, ci, v = random_crs(rng, 60, 500)
        x = rng.uniform(-1, 1, n)
        want = dense_matvec(n, rp, ci, v, x)
        assert max_rel_error(port.spmv_crs(n, rp, ci, v, x), want) <= 1e-10


def test_port_against_live_reference(port, ref):
    rng = np.random.default_rng(4242)
    for _ in range(10):
        n, rp, ci, v = random_crs(rng, 80, 900)
        h = ref.matrix(n, rp, ci, v)
        rc, ell, msg = ref.convert(h, 4)
        assert rc == 0, msg
        bc, ev, ec, cnt = port.crs_to_ell(n, rp, ci, v)
        assert ev.tobytes() == ref.array(ell, 0).tobytes()
        np.testing.assert_array_equal(ec, ref.array(ell, 3))
        if v.shape[0]:
            assert port.row_stats(n, rp) == ref.row_stats(h)
        ref.free(ell)
        ref.free(h)
    # stats: Welford (port) vs the reference on 100 histograms (acceptance.cpp:140-167)
    for _ in range(30):
        counts = rng.integers(0, 1000, size=int(rng.integers(1, 5000)))
        if counts.sum() == 0:
            counts[0] = 1
        rp = np.concatenate([[1], 1 + np.cumsum(counts)])
        assert port.row_stats(len(counts), rp) == ref.stats_from_counts(counts)


def test_find_d_star_brute_force(port, ref):
    rng = np.random.default_rng(71)
    for _ in range(300):
        size = int(rng.integers(0, 50))
        recs = [(6.0 * rng.random(), 5.0 * rng.random()) for _ in range(size)]
        prev = np.inf
        for c in (0.5, 1.0, 2.0):
            got = port.find_d_star(recs, c)
            best = 0.0
            for cand, _ in recs:
                if all(not (d <= cand and r < c) for d, r in recs):
                    best = max(best, cand)
            assert got == best == ref.find_d_star(recs, c)
            assert got <= prev
            prev = got


def test_reference_arm_generator_matches_the_product_generator():
    """bench.py --impl reference builds its matrix inside oracle/_ref (the
    generator compiled there); it must equal the product's byte for byte."""
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built")
    from paper_2407_00019_b200 import spmvtk as sp
    ref = Ref()
    for cfg, param, dparam in ((1, 16, 0.0), (2, 4096, 0.0), (3, 8, 0.0), (4, 8192, 0.0),
                               (5, 4096, 0.7)):
        h = ref.gen_baseline(cfg, param, dparam, 11)
        hc = sp.HostCrs(cfg, param, dparam, 11)
        rp, ci, v = hc.arrays(1)
        assert np.array_equal(ref.array(h, 1), rp), cfg
        assert np.array_equal(ref.array(h, 3), ci), cfg
        assert ref.array(h, 0).tobytes() == v.tobytes(), cfg
        ref.free(h)
        hc.free()
    assert np.array_equal(ref.gen_vector(1000, 5), sp.gen_vector(1000, 5))


def test_ell_bands_are_slices_of_crs_to_ell(port, golden):
    """or_crs_to_ell_bands (band-range ELL for arrays too large to hold at
    once) equals the band slices of the pinned crs_to_ell."""
    for name in sorted(k for k in golden.files if k.endswith("_row_ptr"))[:8]:
        pre = name[: -len("_row_ptr")]
        rp, ci, v = golden[pre + "_row_ptr"], golden[pre + "_col_idx"], golden[pre + "_values"]
        n = rp.shape[0] - 1
        bc, ev, ec, _ = port.crs_to_ell(n, rp, ci, v)
        for k0, k1 in ((1, bc + 1), (1, 2), (max(1, bc // 2), bc + 1)):
            if k1 <= k0:
                continue
            vv, cc = port.crs_to_ell_bands(n, rp, ci, v, k0, k1)
            assert vv.tobytes() == ev[(k0 - 1) * n:(k1 - 1) * n].tobytes()
            np.testing.assert_array_equal(cc, ec[(k0 - 1) * n:(k1 - 1) * n])
