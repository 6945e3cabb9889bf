"""Oracle bindings -- TEST INFRASTRUCTURE ONLY.

Two checkers, both CPU:

* ``Port`` -- ctypes over ``oracle/liboracle.so``, the plain-C restatement of
  the reference algorithms (``oracle/spmvtk_oracle.c``), 1-based int64 arrays
  exactly as the reference lays them out.
* ``Ref`` -- ctypes over ``oracle/_ref/libspmvtk_ref.so``, the reference
  itself compiled from /root/reference/proj/src (``oracle/Makefile``) plus
  ``ref_shim.cpp`` for array in/out and the reference timing protocol.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
CPU baseline; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libspmvtk_ref.so")

_P = C.c_void_p
_i64 = C.c_int64
_pi = C.POINTER(C.c_int64)
_pd = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    """Compiles the C port (always) and the reference (when its sources are
    present, i.e. in the build container)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True, capture_output=True)


def _i(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Port:
    """The plain-C restatement (1-based int64 arrays)."""

    def __init__(self, path: str = PORT_LIB):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_row_stats.argtypes = [_i64, _P, _pd, _pd, _pd]
        L.or_max_row.argtypes = [_i64, _P]
        L.or_max_row.restype = _i64
        L.or_estimate_ell_bytes.argtypes = [_i64, _P, C.c_int, C.c_int]
        L.or_estimate_ell_bytes.restype = C.c_uint64
        for f in ("or_crs_to_coo_row", "or_crs_to_ccs", "or_ccs_to_coo_col"):
            getattr(L, f).argtypes = [_i64, _P, _P, _P, _P, _P, _P]
        L.or_crs_to_ell.argtypes = [_i64, _P, _P, _P, C.c_uint64, _i64, _P, _P, _P]
        L.or_ell_to_rowmajor.argtypes = [_i64, _i64, _P, _P, _P, _P]
        L.or_crs_to_ell_bands.argtypes = [_i64, _P, _P, _P, _i64, _i64, _P, _P]
        L.or_partition_range.argtypes = [_i64, C.c_int, _P, _P]
        L.or_reduce_partials.argtypes = [_i64, C.c_int, _P, _P]
        L.or_spmv_crs.argtypes = [_i64, _P, _P, _P, _P, _P]
        L.or_spmv_coo_outer.argtypes = [_i64, _i64, _P, _P, _P, _P, C.c_int, _P]
        L.or_spmv_ell_inner.argtypes = [_i64, _i64, _P, _P, _P, _P]
        L.or_spmv_ell_outer.argtypes = [_i64, _i64, _P, _P, _P, C.c_int, _P]
        L.or_compute_metrics.argtypes = [C.c_double] * 3 + [_pd] * 3
        L.or_amortization.argtypes = [C.c_double] * 3
        L.or_amortization.restype = C.c_int64
        L.or_find_d_star.argtypes = [C.c_size_t, _P, _P, C.c_double]
        L.or_find_d_star.restype = C.c_double

    # ---- stats / sizes ---------------------------------------------------
    def row_stats(self, n, row_ptr):
        rp = _i(row_ptr)
        mu, sg, dm = C.c_double(), C.c_double(), C.c_double()
        rc = self.lib.or_row_stats(n, _p(rp), C.byref(mu), C.byref(sg), C.byref(dm))
        if rc:
            raise ValueError("row statistics undefined for an empty matrix (mu = 0)")
        return mu.value, sg.value, dm.value

    def max_row(self, n, row_ptr):
        return self.lib.or_max_row(n, _p(_i(row_ptr)))

    def estimate_ell_bytes(self, n, row_ptr, vb=8, ib=8):
        return self.lib.or_estimate_ell_bytes(n, _p(_i(row_ptr)), vb, ib)

    # ---- transforms --------------------------------------------------------
    def crs_to_coo_row(self, n, row_ptr, col_idx, values):
        rp, ci, v = _i(row_ptr), _i(col_idx), _f(values)
        nnz = v.shape[0]
        r, c, vv = np.empty(nnz, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        self.lib.or_crs_to_coo_row(n, _p(rp), _p(ci), _p(v), _p(r), _p(c), _p(vv))
        return r, c, vv

    def crs_to_ccs(self, n, row_ptr, col_idx, values):
        rp, ci, v = _i(row_ptr), _i(col_idx), _f(values)
        nnz = v.shape[0]
        cp, ri, vv = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        self.lib.or_crs_to_ccs(n, _p(rp), _p(ci), _p(v), _p(cp), _p(ri), _p(vv))
        return cp, ri, vv

    def ccs_to_coo_col(self, n, col_ptr, row_idx, values):
        cp, ri, v = _i(col_ptr), _i(row_idx), _f(values)
        nnz = v.shape[0]
        r, c, vv = np.empty(nnz, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        self.lib.or_ccs_to_coo_col(n, _p(cp), _p(ri), _p(v), _p(r), _p(c), _p(vv))
        return r, c, vv

    def crs_to_coo_col(self, n, row_ptr, col_idx, values):
        return self.ccs_to_coo_col(n, *self.crs_to_ccs(n, row_ptr, col_idx, values))

    def crs_to_ell(self, n, row_ptr, col_idx, values, max_bytes=0):
        """-> (band_count, values[n*bc], col_idx[n*bc], row_entry_count[n]) or
        raises MemoryError on the guard (convert.cpp:82-88)."""
        rp, ci, v = _i(row_ptr), _i(col_idx), _f(values)
        bc = self.max_row(n, rp)
        vv = np.empty(n * bc)
        cc = np.empty(n * bc, np.int64)
        cnt = np.empty(n, np.int64)
        rc = self.lib.or_crs_to_ell(n, _p(rp), _p(ci), _p(v), max_bytes, bc, _p(vv), _p(cc),
                                    _p(cnt))
        if rc == 4:
            est = self.estimate_ell_bytes(n, rp)
            raise MemoryError(f"ELL footprint estimate {est} bytes exceeds limit {max_bytes}")
        return bc, vv, cc, cnt

    def crs_to_ell_bands(self, n, row_ptr, col_idx, values, k0, k1):
        """Bands [k0, k1) (1-based) of crs_to_ell: ((k1-k0)*n values, columns)."""
        rp, ci, v = _i(row_ptr), _i(col_idx), _f(values)
        vv = np.empty((k1 - k0) * n)
        cc = np.empty((k1 - k0) * n, np.int64)
        self.lib.or_crs_to_ell_bands(n, _p(rp), _p(ci), _p(v), k0, k1, _p(vv), _p(cc))
        return vv, cc

    def ell_to_rowmajor(self, n, bc, values, col_idx):
        v, c = _f(values), _i(col_idx)
        rv, rc = np.empty(n * bc), np.empty(n * bc, np.int64)
        self.lib.or_ell_to_rowmajor(n, bc, _p(v), _p(c), _p(rv), _p(rc))
        return rv, rc

    # ---- SpMV ----------------------------------------------------------------
    def spmv_crs(self, n, row_ptr, col_idx, values, x):
        y = np.empty(n)
        self.lib.or_spmv_crs(n, _p(_i(row_ptr)), _p(_i(col_idx)), _p(_f(values)), _p(_f(x)),
                             _p(y))
        return y

    def spmv_coo(self, n, row, col, values, x, lanes=1):
        y = np.empty(n)
        v = _f(values)
        self.lib.or_spmv_coo_outer(n, v.shape[0], _p(_i(row)), _p(_i(col)), _p(v), _p(_f(x)),
                                   lanes, _p(y))
        return y

    def spmv_ell_inner(self, n, bc, values, col_idx, x):
        y = np.empty(n)
        self.lib.or_spmv_ell_inner(n, bc, _p(_f(values)), _p(_i(col_idx)), _p(_f(x)), _p(y))
        return y

    def spmv_ell_outer(self, n, bc, values, col_idx, x, lanes=1):
        y = np.empty(n)
        self.lib.or_spmv_ell_outer(n, bc, _p(_f(values)), _p(_i(col_idx)), _p(_f(x)), lanes,
                                   _p(y))
        return y

    # ---- autotune arithmetic -------------------------------------------------
    def gen_baseline(self, config: int, param: int, dparam: float = 0.0, seed: int = 2407):
        """A BASELINE workload as a reference CRS handle (the product's
        generator compiled into this library: no product .so is loaded)."""
        h = C.c_void_p()
        if self.lib.ref_gen_baseline(config, param, float(dparam), seed, C.byref(h)):
            raise RuntimeError(self.err())
        return h

    def gen_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.ref_gen_vector(n, seed, _p(out)):
            raise RuntimeError(self.err())
        return out

    def partition_range(self, length, lanes):
        s, e = np.empty(max(lanes, 1), np.int64), np.empty(max(lanes, 1), np.int64)
        if self.lib.or_partition_range(length, lanes, _p(s), _p(e)):
            raise ValueError("lane count must be at least 1")
        return s, e

    def compute_metrics(self, t_crs, t_ell, t_trans):
        sp, tt, r = C.c_double(), C.c_double(), C.c_double()
        if self.lib.or_compute_metrics(t_crs, t_ell, t_trans, C.byref(sp), C.byref(tt),
                                       C.byref(r)):
            raise ValueError("timings must be positive")
        return sp.value, tt.value, r.value

    def amortization(self, t_crs, t_ell, t_trans):
        k = self.lib.or_amortization(t_crs, t_ell, t_trans)
        if k == -2:
            raise ValueError("timings must be positive")
        return None if k == -1 else k

    def find_d_star(self, records, c):
        d = _f([a for a, _ in records] or [0.0])
        r = _f([b for _, b in records] or [0.0])
        return self.lib.or_find_d_star(len(records), _p(d), _p(r), c)


class Ref:
    """The reference library itself (its C ABI + ref_shim.cpp)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (build with `make -C oracle ref`)")
        self.lib = C.CDLL(path, mode=os.RTLD_LOCAL)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.spmvtk_last_error.restype = C.c_char_p
        L.ref_matrix_from_crs.argtypes = [_i64, _P, _P, _P, C.POINTER(_P)]
        L.ref_matrix_meta.argtypes = [_P, _P]
        L.ref_matrix_get_array.argtypes = [_P, C.c_int, _P, _pi]
        L.ref_measure_spmv.argtypes = [_P, C.c_int, C.c_int, C.c_int, _pd]
        L.ref_measure_transformation.argtypes = [_P, C.c_int, C.c_uint64, _pd, C.POINTER(_P)]
        L.ref_row_stats.argtypes = [_P, _pd, _pd, _pd]
        L.ref_stats_from_counts.argtypes = [_i64, _P, _pd, _pd, _pd]
        L.ref_estimate_ell_bytes.argtypes = [_P, C.c_int, C.c_int]
        L.ref_estimate_ell_bytes.restype = C.c_uint64
        L.ref_find_d_star.argtypes = [C.c_size_t, _P, _P, C.c_double]
        L.ref_find_d_star.restype = C.c_double
        L.ref_amortization.argtypes = [C.c_double] * 3
        L.ref_amortization.restype = C.c_int64
        L.ref_partition_range.argtypes = [_i64, C.c_int, _P, _P]
        L.ref_gen_baseline.argtypes = [C.c_int, _i64, C.c_double, C.c_uint64, C.POINTER(_P)]
        L.ref_gen_vector.argtypes = [_i64, C.c_uint64, _P]
        L.spmvtk_matrix_free.argtypes = [_P]
        L.spmvtk_matrix_convert.argtypes = [_P, C.c_int, C.c_uint64, C.POINTER(_P)]
        L.spmvtk_spmv.argtypes = [_P, C.c_int, _P, _i64, C.c_int, _P, _pd]
        L.spmvtk_gen_banded.argtypes = [_i64, _i64, C.POINTER(_P)]
        L.spmvtk_gen_skewed.argtypes = [_i64, _i64, _i64, _i64, C.c_uint64, C.POINTER(_P)]
        L.spmvtk_gen_cv_target.argtypes = [_i64, C.c_double, C.c_double, C.c_uint64,
                                           C.POINTER(_P)]
        L.spmvtk_matrix_get_format.argtypes = [_P]
        L.spmvtk_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(_P)]
        L.spmvtk_write_matrix_market.argtypes = [_P, C.c_char_p]

    def read_matrix_market(self, path: str):
        """The reference parser: (status, message, handle or None)."""
        h = C.c_void_p()
        st = self.lib.spmvtk_read_matrix_market(str(path).encode(), C.byref(h))
        msg = (self.lib.spmvtk_last_error() or b"").decode()
        return st, msg, (h if st == 0 else None)

    def err(self) -> str:
        return (self.lib.ref_last_error() or b"").decode()

    def matrix(self, n, row_ptr, col_idx, values) -> C.c_void_p:
        rp, ci, v = _i(row_ptr), _i(col_idx), _f(values)
        h = C.c_void_p()
        if self.lib.ref_matrix_from_crs(n, _p(rp), _p(ci), _p(v), C.byref(h)):
            raise RuntimeError(self.err())
        return h

    def free(self, h) -> None:
        self.lib.spmvtk_matrix_free(h)

    def gen(self, kind: str, *args) -> C.c_void_p:
        h = C.c_void_p()
        rc = getattr(self.lib, f"spmvtk_gen_{kind}")(*args, C.byref(h))
        if rc:
            raise RuntimeError(self.lib.spmvtk_last_error().decode())
        return h

    def meta(self, h) -> dict:
        m = np.zeros(5, np.int64)
        self.lib.ref_matrix_meta(h, _p(m))
        return {"n": int(m[0]), "nnz": int(m[1]), "band_count": int(m[2]),
                "stored_nnz": int(m[3]), "ordering": int(m[4])}

    def array(self, h, which: int) -> np.ndarray:
        n = _i64()
        if self.lib.ref_matrix_get_array(h, which, None, C.byref(n)):
            raise RuntimeError(self.err())
        out = np.empty(n.value, np.float64 if which == 0 else np.int64)
        self.lib.ref_matrix_get_array(h, which, _p(out), C.byref(n))
        return out

    def convert(self, h, fmt: int, max_bytes: int = 0):
        out = C.c_void_p()
        rc = self.lib.spmvtk_matrix_convert(h, fmt, max_bytes, C.byref(out))
        return rc, out, self.lib.spmvtk_last_error().decode()

    def spmv(self, h, kernel: int, x, lanes: int = 1):
        xs = _f(x)
        y = np.empty_like(xs)
        el = C.c_double()
        rc = self.lib.spmvtk_spmv(h, kernel, _p(xs), xs.shape[0], lanes, _p(y), C.byref(el))
        if rc:
            raise RuntimeError(self.lib.spmvtk_last_error().decode())
        return y, el.value

    def measure_spmv(self, h, kernel: int, lanes: int, repeats: int) -> float:
        s = C.c_double()
        if self.lib.ref_measure_spmv(h, kernel, lanes, repeats, C.byref(s)):
            raise RuntimeError(self.err())
        return s.value

    def measure_transformation(self, h, fmt: int, max_bytes: int = 0):
        s = C.c_double()
        out = C.c_void_p()
        rc = self.lib.ref_measure_transformation(h, fmt, max_bytes, C.byref(s), C.byref(out))
        if rc:
            raise RuntimeError(self.err())
        return s.value, out

    def row_stats(self, h):
        mu, sg, dm = C.c_double(), C.c_double(), C.c_double()
        if self.lib.ref_row_stats(h, C.byref(mu), C.byref(sg), C.byref(dm)):
            raise ValueError(self.err())
        return mu.value, sg.value, dm.value

    def stats_from_counts(self, counts):
        c = _i(counts)
        mu, sg, dm = C.c_double(), C.c_double(), C.c_double()
        if self.lib.ref_stats_from_counts(c.shape[0], _p(c), C.byref(mu), C.byref(sg),
                                          C.byref(dm)):
            raise ValueError(self.err())
        return mu.value, sg.value, dm.value

    def find_d_star(self, records, c):
        d = _f([a for a, _ in records] or [0.0])
        r = _f([b for _, b in records] or [0.0])
        return self.lib.ref_find_d_star(len(records), _p(d), _p(r), c)

    def amortization(self, t_crs, t_ell, t_trans):
        k = self.lib.ref_amortization(t_crs, t_ell, t_trans)
        return None if k == -1 else k

    def gen_baseline(self, config: int, param: int, dparam: float = 0.0, seed: int = 2407):
        """A BASELINE workload as a reference CRS handle (the product's
        generator compiled into this library: no product .so is loaded)."""
        h = C.c_void_p()
        if self.lib.ref_gen_baseline(config, param, float(dparam), seed, C.byref(h)):
            raise RuntimeError(self.err())
        return h

    def gen_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.ref_gen_vector(n, seed, _p(out)):
            raise RuntimeError(self.err())
        return out

    def partition_range(self, length, lanes):
        s, e = np.empty(max(lanes, 1), np.int64), np.empty(max(lanes, 1), np.int64)
        if self.lib.ref_partition_range(length, lanes, _p(s), _p(e)):
            raise ValueError(self.err())
        return s, e


def random_crs(rng: np.random.Generator, max_n: int, max_nnz: int, sorted_cols=False):
    """Random square CRS with distinct positions and (by default) UNSORTED
    columns inside rows, values U[-1,1) -- the shape of the reference's
    test_support.hpp:43-74 generator (numpy RNG here).  1-based int64."""
    n = int(rng.integers(1, max_n + 1))
    want = int(rng.integers(0, min(max_nnz, n * n) + 1))
    flat = rng.choice(n * n, size=want, replace=False) if want else np.empty(0, np.int64)
    rows = flat // n
    cols = flat % n
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    vals = rng.uniform(-1.0, 1.0, size=want)
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr) + 1
    if not sorted_cols:
        for i in range(n):
            a, b = row_ptr[i] - 1, row_ptr[i + 1] - 1
            if b - a > 1:
                p = rng.permutation(b - a) + a
                cols[a:b] = cols[p]
                vals[a:b] = vals[p]
    return n, row_ptr, cols + 1, vals


def dense_matvec(n, row_ptr, col_idx, values, x):
    d = np.zeros((n, n))
    for i in range(n):
        for p in range(row_ptr[i] - 1, row_ptr[i + 1] - 1):
            d[i, col_idx[p] - 1] = values[p]
    return d @ np.asarray(x, dtype=np.float64)


def max_rel_error(got, want) -> float:
    """max|g - w| / max|w| (test_support.hpp:96-105)."""
    got = np.asarray(got)
    want = np.asarray(want)
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    if scale == 0.0:
        scale = 1.0
    return float(np.max(np.abs(got - want)) / scale) if got.size else 0.0
