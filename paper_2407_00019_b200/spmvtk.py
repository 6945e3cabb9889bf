"""Python binding of the spmvtk C ABI (``include/spmvtk/spmvtk.h``).

A thin ctypes layer over ``libspmvtk.so``: the work happens in the sm_100a
kernels behind the C ABI; this module only marshals arrays and maps status
codes to exceptions.  It mirrors the reference's C API
(/root/reference/proj/include/spmvtk/spmvtk.h:50-160) one function per entry
point, with the same enum values and error mapping, so the tests read like
the reference's ``test_capi.cpp``.

There is no CPU fallback: importing works without a GPU (so the CPU test
suite can check that the library loads and exports every symbol), but any
call that needs the device fails with the CUDA error surfaced as
``SpmvtkError``.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPMVTK_LIBRARY: another build of the same library (A/B timing in tools/)
LIB_PATH = os.environ.get("SPMVTK_LIBRARY") or os.path.join(_HERE, "libspmvtk.so")


class Status(enum.IntEnum):
    OK = 0
    ERR_USAGE = 1
    ERR_DATA = 2
    ERR_CHECK = 3
    ERR_MEMORY_LIMIT = 4


class Format(enum.IntEnum):
    CRS = 0
    CCS = 1
    COO_ROW = 2
    COO_COL = 3
    ELL = 4
    ELL_ROWMAJOR = 5


class Kernel(enum.IntEnum):
    CRS = 0
    COO_ROW_OUTER = 1
    COO_COL_OUTER = 2
    ELL_INNER = 3
    ELL_OUTER = 4
    ELL_ROWMAJOR = 5


class Decision(enum.IntEnum):
    USE_ELL = 0
    USE_CRS = 1


class Array(enum.IntEnum):
    VALUES = 0
    POINTER = 1
    ROW_IDX = 2
    COL_IDX = 3
    ROW_ENTRY_COUNT = 4


KERNEL_NAMES = {
    Kernel.CRS: "crs",
    Kernel.COO_ROW_OUTER: "coo-row",
    Kernel.COO_COL_OUTER: "coo-col",
    Kernel.ELL_INNER: "ell-inner",
    Kernel.ELL_OUTER: "ell-outer",
    Kernel.ELL_ROWMAJOR: "ell-row",
}

# kernel -> the format its handle must have
KERNEL_FORMAT = {
    Kernel.CRS: Format.CRS,
    Kernel.COO_ROW_OUTER: Format.COO_ROW,
    Kernel.COO_COL_OUTER: Format.COO_COL,
    Kernel.ELL_INNER: Format.ELL,
    Kernel.ELL_OUTER: Format.ELL,
    Kernel.ELL_ROWMAJOR: Format.ELL_ROWMAJOR,
}


class SpmvtkError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{Status(status).name}: {message}")
        self.status = Status(status)
        self.message = message


class MatrixInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("max_row_entries", C.c_int64),
                ("mu", C.c_double), ("sigma", C.c_double), ("d_mat", C.c_double),
                ("ell_bytes", C.c_uint64)]


class BenchResult(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("t_crs", "t_ell", "t_trans", "sp", "tt", "r")]


class RecordView(C.Structure):
    _fields_ = [("matrix_id", C.c_char_p), ("n", C.c_int64), ("nnz", C.c_int64),
                ("mu", C.c_double), ("sigma", C.c_double), ("d_mat", C.c_double),
                ("excluded", C.c_int), ("exclusion_reason", C.c_char_p),
                ("t_crs", C.c_double), ("t_ell", C.c_double), ("t_trans", C.c_double),
                ("sp", C.c_double), ("tt", C.c_double), ("r", C.c_double)]


class MatrixDesc(C.Structure):
    _fields_ = [("format", C.c_int32), ("ordering", C.c_int32), ("n", C.c_int64),
                ("nnz", C.c_int64), ("band_count", C.c_int64), ("ld", C.c_int64),
                ("device_bytes", C.c_uint64), ("ncols", C.c_int64), ("row_offset", C.c_int64)]


MAX_PEERS = 8
IPC_HANDLE_BYTES = 64


class Push(C.Structure):
    """spmvtk_push: destinations of pushed result rows (spmvtk.h)."""
    _fields_ = [("dst", C.c_void_p * MAX_PEERS), ("mask", C.c_void_p), ("ndst", C.c_int32),
                ("local", C.c_int32)]


class FlagTargets(C.Structure):
    """spmvtk_flag_targets: this rank's flag slot in every peer's array."""
    _fields_ = [("ptr", C.c_void_p * MAX_PEERS), ("n", C.c_int32)]


class PushSync(C.Structure):
    """spmvtk_push_sync: the step's flag wait / signal inside the SpMV launch."""
    _fields_ = [("wait_flags", C.c_void_p), ("nwait", C.c_int32), ("wait_value", C.c_uint64),
                ("timeout_ns", C.c_uint64), ("status", C.c_void_p), ("signal", FlagTargets),
                ("signal_value", C.c_uint64), ("counter", C.c_void_p)]


class RowStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("max_row", C.c_int64),
                ("mu", C.c_double), ("sigma", C.c_double), ("d_mat", C.c_double)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_i64 = C.c_int64
_u64 = C.c_uint64
_d = C.c_double
_pd = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol of spmvtk.h
SIGNATURES = {
    # part 1: the reference ABI
    "spmvtk_last_error": (C.c_char_p, []),
    "spmvtk_matrix_free": (None, [_P]),
    "spmvtk_profile_free": (None, [_P]),
    "spmvtk_read_matrix_market": (C.c_int, [C.c_char_p, _PP]),
    "spmvtk_write_matrix_market": (C.c_int, [_P, C.c_char_p]),
    "spmvtk_gen_banded": (C.c_int, [_i64, _i64, _PP]),
    "spmvtk_gen_skewed": (C.c_int, [_i64, _i64, _i64, _i64, _u64, _PP]),
    "spmvtk_gen_cv_target": (C.c_int, [_i64, _d, _d, _u64, _PP]),
    "spmvtk_matrix_get_format": (C.c_int, [_P]),
    "spmvtk_matrix_get_info": (C.c_int, [_P, C.POINTER(MatrixInfo)]),
    "spmvtk_matrix_convert": (C.c_int, [_P, C.c_int, _u64, _PP]),
    "spmvtk_matrix_convert_timed": (C.c_int, [_P, C.c_int, _u64, _PP, _pd]),
    "spmvtk_spmv": (C.c_int, [_P, C.c_int, _P, _i64, C.c_int, _P, _pd]),
    "spmvtk_bench": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _u64, C.POINTER(BenchResult)]),
    "spmvtk_profile_build": (C.c_int, [C.POINTER(_P), C.POINTER(C.c_char_p), C.c_size_t, C.c_int,
                                       C.c_int, _d, C.c_int, _u64, C.c_char_p, _PP]),
    "spmvtk_profile_write": (C.c_int, [_P, C.c_char_p]),
    "spmvtk_profile_read": (C.c_int, [C.c_char_p, _PP]),
    "spmvtk_profile_d_star": (_d, [_P]),
    "spmvtk_profile_c": (_d, [_P]),
    "spmvtk_profile_lanes": (C.c_int, [_P]),
    "spmvtk_profile_kernel": (C.c_int, [_P]),
    "spmvtk_profile_record_count": (C.c_size_t, [_P]),
    "spmvtk_profile_record": (C.c_int, [_P, C.c_size_t, C.POINTER(RecordView)]),
    "spmvtk_select": (C.c_int, [_P, _P, C.POINTER(C.c_int), _pd]),
    # part 2: extensions
    "spmvtk_set_stream": (None, [_P]),
    "spmvtk_get_stream": (_P, []),
    "spmvtk_synchronize": (C.c_int, []),
    "spmvtk_matrix_from_crs": (C.c_int, [_i64, _i64, _P, _P, _P, C.c_int, C.c_int, C.c_int, _PP]),
    "spmvtk_matrix_from_crs_block": (C.c_int, [_i64, _i64, _i64, _i64, _P, _P, _P, C.c_int,
                                               C.c_int, C.c_int, _PP]),
    "spmvtk_matrix_to_crs": (C.c_int, [_P, _PP]),
    "spmvtk_matrix_describe": (C.c_int, [_P, C.POINTER(MatrixDesc)]),
    "spmvtk_matrix_copy_array": (C.c_int, [_P, C.c_int, _P, _i64, C.c_int, C.c_int,
                                           C.POINTER(_i64)]),
    "spmvtk_matrix_device_array": (C.c_int, [_P, C.c_int, _PP, C.POINTER(_i64)]),
    "spmvtk_spmv_device": (C.c_int, [_P, C.c_int, _P, _P]),
    "spmvtk_matrix_row_stats": (C.c_int, [_P, C.POINTER(RowStats)]),
    "spmvtk_gen_baseline": (C.c_int, [C.c_int, _i64, _d, _u64, _PP]),
    "spmvtk_gen_vector": (C.c_int, [_i64, _u64, _P]),
    "spmvtk_gen_baseline_host": (C.c_int, [C.c_int, _i64, _d, _u64, _PP, C.POINTER(_i64),
                                           C.POINTER(_i64)]),
    "spmvtk_read_matrix_market_host": (C.c_int, [C.c_char_p, _PP, C.POINTER(_i64),
                                                 C.POINTER(_i64)]),
    "spmvtk_host_crs_export": (C.c_int, [_P, _P, _P, _P, C.c_int]),
    "spmvtk_matrix_copy_ell_bands": (C.c_int, [_P, _i64, _i64, _P, _P, C.c_int]),
    "spmvtk_dist_unique_id": (C.c_int, [_P]),
    "spmvtk_dist_init": (C.c_int, [C.c_int, C.c_int, _P, _PP]),
    "spmvtk_dist_free": (None, [_P]),
    "spmvtk_partition_rows": (C.c_int, [_P, _i64, C.c_int, _P]),
    "spmvtk_matrix_distribute": (C.c_int, [_P, _i64, _P, _P, _P, C.c_int, C.c_int, _PP]),
    "spmvtk_gen_baseline_shard_host": (C.c_int, [C.c_int, _i64, _d, _u64, C.c_int, C.c_int, _PP,
                                                 C.POINTER(_i64), C.POINTER(_i64),
                                                 C.POINTER(_i64)]),
    "spmvtk_gen_baseline_shard": (C.c_int, [_P, C.c_int, _i64, _d, _u64, _PP]),
    "spmvtk_dist_spmv_iterate": (C.c_int, [_P, _P, C.c_int, _P, _i64, _pd]),
    "spmvtk_dist_push_create": (C.c_int, [_P, _P, C.c_int, C.c_int, _PP]),
    "spmvtk_dist_push_iterate": (C.c_int, [_P, _P, _i64, _pd]),
    "spmvtk_dist_push_free": (None, [_P]),
    "spmvtk_host_crs_free": (None, [_P]),
    "spmvtk_matrix_from_host_crs": (C.c_int, [_P, _PP]),
    "spmvtk_conversion_bytes": (C.c_int, [_P, C.c_int, C.POINTER(_u64), C.POINTER(_u64)]),
    "spmvtk_transform_kernel_seconds": (C.c_int, [_P, C.c_int, C.c_int, _pd]),
    "spmvtk_reserve_device_memory": (C.c_int, [_u64]),
    "spmvtk_pipeline_create": (C.c_int, [_P, C.c_int, _PP]),
    "spmvtk_pipeline_submit": (C.c_int, [_P, _P, _P]),
    "spmvtk_pipeline_wait": (C.c_int, [_P]),
    "spmvtk_pipeline_free": (None, [_P]),
    "spmvtk_ipc_alloc": (C.c_int, [_u64, _PP, _P]),
    "spmvtk_ipc_free": (C.c_int, [_P]),
    "spmvtk_ipc_open": (C.c_int, [_P, _PP]),
    "spmvtk_ipc_close": (C.c_int, [_P]),
    "spmvtk_spmv_device_push": (C.c_int, [_P, C.c_int, _P, C.POINTER(Push), _P]),
    "spmvtk_flags_signal": (C.c_int, [C.POINTER(FlagTargets), _u64]),
    "spmvtk_flags_wait": (C.c_int, [_P, C.c_int32, _u64, _u64, _P]),
    "spmvtk_compute_metrics": (C.c_int, [_d, _d, _d, _pd, _pd, _pd]),
    "spmvtk_amortization_iterations": (C.c_int, [_d, _d, _d, C.POINTER(_i64)]),
    "spmvtk_find_d_star": (_d, [_pd, _pd, C.c_size_t, _d]),
    "spmvtk_version": (C.c_char_p, []),
    # lower C ABI (device pointers); only the tuning knob is used from Python
    "spmvtk_k_tune": (C.c_int, [C.c_char_p, C.c_int]),
    "spmvtk_k_gather_probe": (C.c_int, [_P, _i64, C.c_int, _P, _P]),
}

_lib: C.CDLL | None = None


def load_library(path: str | None = None) -> C.CDLL:
    """Loads libspmvtk.so (RTLD_LOCAL) and declares every entry point.

    Raises FileNotFoundError when the native library has not been built --
    there is no Python fallback for the compute path."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise FileNotFoundError(
            f"{p} missing: build it with `python -m paper_2407_00019_b200.build` "
            "(the CUDA path has no fallback)")
    lib = C.CDLL(p, mode=os.RTLD_LOCAL | os.RTLD_NOW)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def _check(status: int, lib: C.CDLL | None = None) -> None:
    if status != 0:
        lib = lib or load_library()
        raise SpmvtkError(status, lib.spmvtk_last_error().decode())


def last_error() -> str:
    return load_library().spmvtk_last_error().decode()


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def set_stream(stream_handle: int | None) -> None:
    """Routes this thread's GPU work to a cudaStream_t (e.g.
    ``torch.cuda.current_stream().cuda_stream``)."""
    load_library().spmvtk_set_stream(C.c_void_p(stream_handle or 0))


def synchronize() -> None:
    _check(load_library().spmvtk_synchronize())


class Matrix:
    """Owning wrapper of a ``spmvtk_matrix*`` (device-resident)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        self._lib = load_library()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def free(self) -> None:
        if self._h:
            self._lib.spmvtk_matrix_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.free()
        except Exception:
            pass

    # ---- constructors -------------------------------------------------
    @staticmethod
    def _make(fn, *args) -> "Matrix":
        out = C.c_void_p()
        _check(fn(*args, C.byref(out)))
        return Matrix(out)

    @classmethod
    def from_crs(cls, n: int, row_ptr, col_idx, values, index_base: int = 0) -> "Matrix":
        rp = np.ascontiguousarray(row_ptr)
        ci = np.ascontiguousarray(col_idx)
        if rp.dtype not in (np.int32, np.int64):
            rp = rp.astype(np.int64)
        ci = ci.astype(rp.dtype, copy=False)
        v = np.ascontiguousarray(values, dtype=np.float64)
        nnz = int(v.shape[0])
        lib = load_library()
        return cls._make(lib.spmvtk_matrix_from_crs, n, nnz, _ptr(rp), _ptr(ci), _ptr(v),
                         rp.dtype.itemsize, index_base, 0)

    @classmethod
    def from_crs_block(cls, nrows: int, ncols: int, row_offset: int, row_ptr, col_idx, values,
                       index_base: int = 0) -> "Matrix":
        """Row-block shard (multi-GPU): local rows, global columns."""
        rp = np.ascontiguousarray(row_ptr)
        if rp.dtype not in (np.int32, np.int64):
            rp = rp.astype(np.int64)
        ci = np.ascontiguousarray(col_idx).astype(rp.dtype, copy=False)
        v = np.ascontiguousarray(values, dtype=np.float64)
        lib = load_library()
        return cls._make(lib.spmvtk_matrix_from_crs_block, nrows, ncols, row_offset,
                         int(v.shape[0]), _ptr(rp), _ptr(ci), _ptr(v), rp.dtype.itemsize,
                         index_base, 0)

    @classmethod
    def from_crs_device(cls, n: int, nnz: int, row_ptr_ptr: int, col_idx_ptr: int,
                        values_ptr: int, index_width: int = 4, index_base: int = 0) -> "Matrix":
        lib = load_library()
        return cls._make(lib.spmvtk_matrix_from_crs, n, nnz, C.c_void_p(row_ptr_ptr),
                         C.c_void_p(col_idx_ptr), C.c_void_p(values_ptr), index_width,
                         index_base, 1)

    @classmethod
    def gen_banded(cls, n: int, half_width: int) -> "Matrix":
        return cls._make(load_library().spmvtk_gen_banded, n, half_width)

    @classmethod
    def gen_skewed(cls, n, base_deg, heavy_rows, heavy_deg, seed=0) -> "Matrix":
        return cls._make(load_library().spmvtk_gen_skewed, n, base_deg, heavy_rows,
                         heavy_deg, seed)

    @classmethod
    def gen_cv_target(cls, n, mean_deg, target_dmat, seed=0) -> "Matrix":
        return cls._make(load_library().spmvtk_gen_cv_target, n, float(mean_deg),
                         float(target_dmat), seed)

    @classmethod
    def gen_baseline(cls, config: int, param: int, dparam: float = 0.0,
                     seed: int = 2407) -> "Matrix":
        return cls._make(load_library().spmvtk_gen_baseline, config, param, float(dparam), seed)

    @classmethod
    def read_matrix_market(cls, path: str) -> "Matrix":
        return cls._make(load_library().spmvtk_read_matrix_market, path.encode())

    # ---- inspection ---------------------------------------------------
    @property
    def format(self) -> Format:
        return Format(self._lib.spmvtk_matrix_get_format(self._h))

    def info(self) -> MatrixInfo:
        out = MatrixInfo()
        _check(self._lib.spmvtk_matrix_get_info(self._h, C.byref(out)))
        return out

    def describe(self) -> MatrixDesc:
        out = MatrixDesc()
        _check(self._lib.spmvtk_matrix_describe(self._h, C.byref(out)))
        return out

    def row_stats(self) -> RowStats:
        out = RowStats()
        _check(self._lib.spmvtk_matrix_row_stats(self._h, C.byref(out)))
        return out

    def array(self, which: Array, index_width: int = 8, index_base: int = 1) -> np.ndarray:
        n = _i64()
        _check(self._lib.spmvtk_matrix_copy_array(self._h, int(which), None, 0, index_width,
                                                  index_base, C.byref(n)))
        dt = np.float64 if which == Array.VALUES else (np.int64 if index_width == 8 else np.int32)
        out = np.empty(n.value, dtype=dt)
        _check(self._lib.spmvtk_matrix_copy_array(self._h, int(which), _ptr(out), n.value,
                                                  index_width, index_base, C.byref(n)))
        return out

    def device_array(self, which: Array) -> tuple[int, int]:
        p = C.c_void_p()
        n = _i64()
        _check(self._lib.spmvtk_matrix_device_array(self._h, int(which), C.byref(p), C.byref(n)))
        return (p.value or 0), n.value

    def conversion_bytes(self, to: Format) -> tuple[int, int]:
        a, b = _u64(), _u64()
        _check(self._lib.spmvtk_conversion_bytes(self._h, int(to), C.byref(a), C.byref(b)))
        return a.value, b.value

    # ---- operations ---------------------------------------------------
    def convert(self, to: Format, max_bytes: int = 0) -> "Matrix":
        return Matrix._make(self._lib.spmvtk_matrix_convert, self._h, int(to), max_bytes)

    def convert_timed(self, to: Format, max_bytes: int = 0) -> tuple["Matrix", float]:
        """convert() timed inside the library as the reference's
        measure_transformation: (handle, t_trans seconds)."""
        out, s = C.c_void_p(), C.c_double()
        _check(self._lib.spmvtk_matrix_convert_timed(self._h, int(to), max_bytes, C.byref(out),
                                                     C.byref(s)))
        return Matrix(out), s.value

    def to_crs(self) -> "Matrix":
        """Canonical CRS rebuilt on the device (inverse conversions)."""
        return Matrix._make(self._lib.spmvtk_matrix_to_crs, self._h)

    def spmv(self, x, kernel: Kernel = Kernel.CRS, lanes: int = 1,
             out: np.ndarray | None = None) -> tuple[np.ndarray, float]:
        xs = np.ascontiguousarray(x, dtype=np.float64)
        # y has one entry per row (== len(x) except for row-block shards)
        nrows = self.describe().n
        if out is not None:
            if not (isinstance(out, np.ndarray) and out.dtype == np.float64
                    and out.flags.c_contiguous and out.shape == (nrows,)):
                raise ValueError(f"out must be a contiguous float64 array of {nrows} rows")
            y = out
        else:
            y = np.empty(nrows, dtype=np.float64)
        el = C.c_double()
        _check(self._lib.spmvtk_spmv(self._h, int(kernel), _ptr(xs), xs.shape[0], lanes,
                                     _ptr(y), C.byref(el)))
        return y, el.value

    def ell_bands(self, k0: int, k1: int, index_base: int = 1):
        """Bands [k0, k1) (0-based) of a band-major ELL: (values, columns)."""
        n = self.describe().n
        v = np.empty((k1 - k0) * n)
        c = np.empty((k1 - k0) * n, np.int64)
        _check(self._lib.spmvtk_matrix_copy_ell_bands(self._h, k0, k1, _ptr(v), _ptr(c),
                                                      index_base))
        return v, c

    def spmv_device(self, kernel: Kernel, x_ptr: int, y_ptr: int) -> None:
        _check(self._lib.spmvtk_spmv_device(self._h, int(kernel), C.c_void_p(x_ptr),
                                            C.c_void_p(y_ptr)))

    def spmv_device_push(self, kernel: Kernel, x_ptr: int, push: "Push",
                         sync: "PushSync | None" = None) -> None:
        """SpMV with the result rows stored to push.dst[w] (multi-GPU
        exchange folded into the product; CRS and ELL_INNER); `sync` folds
        the step's flag wait and signal into the same launch."""
        _check(self._lib.spmvtk_spmv_device_push(
            self._h, int(kernel), C.c_void_p(x_ptr), C.byref(push),
            C.cast(C.byref(sync), C.c_void_p) if sync is not None else None))

    def write_matrix_market(self, path: str) -> None:
        _check(self._lib.spmvtk_write_matrix_market(self._h, path.encode()))

    def transform_kernel_seconds(self, to: Format, repeats: int = 5) -> float:
        s = C.c_double()
        _check(self._lib.spmvtk_transform_kernel_seconds(self._h, int(to), repeats, C.byref(s)))
        return s.value


def reserve_device_memory(nbytes: int) -> None:
    _check(load_library().spmvtk_reserve_device_memory(int(nbytes)))


class Pipeline:
    """Streaming host SpMV (spmvtk_pipeline_*): submit() enqueues
    H2D(x) -> SpMV -> D2H(y) and returns; products overlap each other's
    copies.  x / y must be host buffers (numpy, pinned for asynchrony) that
    stay alive and untouched until wait()."""

    def __init__(self, m: "Matrix", kernel: Kernel):
        self._lib = load_library()
        h = C.c_void_p()
        _check(self._lib.spmvtk_pipeline_create(m.handle, int(kernel), C.byref(h)))
        self._h = h.value
        self._m = m  # the C pipeline borrows the handle: keep it alive
        d = m.describe()
        self._ncols, self._nrows = d.ncols, d.n
        self._keep = []

    def submit(self, x: np.ndarray, y: np.ndarray) -> None:
        # the C side takes bare pointers (no lengths): a short buffer would
        # be read / written past its end by the asynchronous copies
        for a, want, name in ((x, self._ncols, "x"), (y, self._nrows, "y")):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64
                    and a.flags.c_contiguous and a.shape == (want,)):
                raise ValueError(f"{name} must be a contiguous float64 array of length {want}")
        self._keep.append((x, y))
        _check(self._lib.spmvtk_pipeline_submit(self._h, x.ctypes.data, y.ctypes.data))

    def wait(self) -> None:
        _check(self._lib.spmvtk_pipeline_wait(self._h))
        self._keep = []

    def free(self) -> None:
        if self._h:
            self._lib.spmvtk_pipeline_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass


def ipc_alloc(nbytes: int) -> tuple[int, bytes]:
    """cudaMalloc'ed, zeroed device buffer + its 64-byte CUDA IPC handle."""
    p = C.c_void_p()
    h = C.create_string_buffer(IPC_HANDLE_BYTES)
    _check(load_library().spmvtk_ipc_alloc(int(nbytes), C.byref(p), h))
    return int(p.value), h.raw


def ipc_free(ptr: int) -> None:
    _check(load_library().spmvtk_ipc_free(C.c_void_p(ptr)))


def ipc_open(handle: bytes) -> int:
    """Maps a peer process's buffer into this process (device pointer)."""
    p = C.c_void_p()
    buf = C.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
    _check(load_library().spmvtk_ipc_open(buf, C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(load_library().spmvtk_ipc_close(C.c_void_p(ptr)))


def flags_signal(targets: "FlagTargets", value: int) -> None:
    _check(load_library().spmvtk_flags_signal(C.byref(targets), int(value)))


def flags_wait(flags_ptr: int, n: int, value: int, timeout_ns: int, status_ptr: int) -> None:
    _check(load_library().spmvtk_flags_wait(C.c_void_p(flags_ptr), int(n), int(value),
                                            int(timeout_ns), C.c_void_p(status_ptr)))


def bench(m: Matrix, variant: Kernel, lanes: int = 1, repeats: int = 9,
          max_bytes: int = 0) -> dict:
    out = BenchResult()
    _check(load_library().spmvtk_bench(m.handle, int(variant), lanes, repeats, max_bytes,
                                       C.byref(out)))
    return {k: getattr(out, k) for k, _ in BenchResult._fields_}


class Profile:
    def __init__(self, handle: C.c_void_p):
        self._h = handle
        self._lib = load_library()

    @classmethod
    def build(cls, matrices: Sequence[Matrix], ids: Sequence[str], variant: Kernel,
              lanes: int = 1, c: float = 1.0, repeats: int = 9, max_bytes: int = 0,
              label: str = "") -> "Profile":
        lib = load_library()
        mats = (C.c_void_p * len(matrices))(*[m.handle for m in matrices])
        cids = (C.c_char_p * len(ids))(*[s.encode() for s in ids])
        out = C.c_void_p()
        _check(lib.spmvtk_profile_build(mats, cids, len(matrices), int(variant), lanes, c,
                                        repeats, max_bytes, label.encode(), C.byref(out)))
        return cls(out)

    @classmethod
    def read(cls, path: str) -> "Profile":
        out = C.c_void_p()
        _check(load_library().spmvtk_profile_read(path.encode(), C.byref(out)))
        return cls(out)

    def write(self, path: str) -> None:
        _check(self._lib.spmvtk_profile_write(self._h, path.encode()))

    @property
    def handle(self):
        return self._h

    @property
    def d_star(self) -> float:
        return self._lib.spmvtk_profile_d_star(self._h)

    @property
    def c(self) -> float:
        return self._lib.spmvtk_profile_c(self._h)

    @property
    def lanes(self) -> int:
        return self._lib.spmvtk_profile_lanes(self._h)

    @property
    def kernel(self) -> Kernel:
        return Kernel(self._lib.spmvtk_profile_kernel(self._h))

    def records(self) -> list[dict]:
        out = []
        for i in range(self._lib.spmvtk_profile_record_count(self._h)):
            v = RecordView()
            _check(self._lib.spmvtk_profile_record(self._h, i, C.byref(v)))
            d = {k: getattr(v, k) for k, _ in RecordView._fields_}
            d["matrix_id"] = v.matrix_id.decode()
            d["exclusion_reason"] = v.exclusion_reason.decode() if v.exclusion_reason else None
            out.append(d)
        return out

    def free(self) -> None:
        if self._h:
            self._lib.spmvtk_profile_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass


def select(m: Matrix, p: Profile) -> tuple[Decision, float]:
    dec = C.c_int()
    dm = C.c_double()
    _check(load_library().spmvtk_select(m.handle, p.handle, C.byref(dec), C.byref(dm)))
    return Decision(dec.value), dm.value


def compute_metrics(t_crs: float, t_ell: float, t_trans: float) -> tuple[float, float, float]:
    sp, tt, r = C.c_double(), C.c_double(), C.c_double()
    _check(load_library().spmvtk_compute_metrics(t_crs, t_ell, t_trans, C.byref(sp),
                                                 C.byref(tt), C.byref(r)))
    return sp.value, tt.value, r.value


def amortization_iterations(t_crs: float, t_ell: float, t_trans: float) -> int | None:
    k = _i64()
    _check(load_library().spmvtk_amortization_iterations(t_crs, t_ell, t_trans, C.byref(k)))
    return None if k.value < 0 else k.value


def find_d_star(records: Iterable[tuple[float, float]], c: float) -> float:
    recs = list(records)
    d = (C.c_double * max(1, len(recs)))(*[a for a, _ in recs])
    r = (C.c_double * max(1, len(recs)))(*[b for _, b in recs])
    return load_library().spmvtk_find_d_star(d, r, len(recs), c)


class HostCrs:
    """A BASELINE workload generated in host memory only (no device)."""

    def __init__(self, config: int, param: int, dparam: float = 0.0, seed: int = 2407):
        self._lib = load_library()
        self._h = C.c_void_p()
        n, nnz = _i64(), _i64()
        _check(self._lib.spmvtk_gen_baseline_host(config, param, float(dparam), seed,
                                                  C.byref(self._h), C.byref(n), C.byref(nnz)))
        self.n, self.nnz = n.value, nnz.value

    @classmethod
    def read_matrix_market(cls, path: str) -> "HostCrs":
        """Matrix Market file -> host CRS (no device work)."""
        self = cls.__new__(cls)
        self._lib = load_library()
        self._h = C.c_void_p()
        n, nnz = _i64(), _i64()
        _check(self._lib.spmvtk_read_matrix_market_host(str(path).encode(), C.byref(self._h),
                                                        C.byref(n), C.byref(nnz)))
        self.n, self.nnz = n.value, nnz.value
        return self

    def arrays(self, index_base: int = 1):
        rp = np.empty(self.n + 1, np.int64)
        ci = np.empty(self.nnz, np.int64)
        v = np.empty(self.nnz, np.float64)
        _check(self._lib.spmvtk_host_crs_export(self._h, _ptr(rp), _ptr(ci), _ptr(v), index_base))
        return rp, ci, v

    def upload(self) -> Matrix:
        return Matrix._make(self._lib.spmvtk_matrix_from_host_crs, self._h)

    def free(self) -> None:
        if self._h:
            self._lib.spmvtk_host_crs_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass


def gen_vector(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(load_library().spmvtk_gen_vector(n, seed, _ptr(out)))
    return out


DIST_ID_BYTES = 128


def partition_rows(row_ptr, world: int) -> np.ndarray:
    """Entry-balanced contiguous row blocks (spmvtk_partition_rows): begin[world+1]."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.empty(world + 1, np.int64)
    _check(load_library().spmvtk_partition_rows(_ptr(rp), rp.shape[0] - 1, world, _ptr(out)))
    return out


def gen_baseline_shard_host(config: int, param: int, dparam: float, seed: int, rank: int,
                            world: int) -> "HostCrs":
    """This rank's row block of a BASELINE workload, generated alone (host)."""
    self = HostCrs.__new__(HostCrs)
    self._lib = load_library()
    self._h = C.c_void_p()
    rows, off, ncols = _i64(), _i64(), _i64()
    _check(self._lib.spmvtk_gen_baseline_shard_host(config, param, float(dparam), seed, rank, world,
                                                    C.byref(self._h), C.byref(rows), C.byref(off),
                                                    C.byref(ncols)))
    self.n = rows.value
    self.row_offset, self.ncols = off.value, ncols.value
    rp = np.empty(self.n + 1, np.int64)
    _check(self._lib.spmvtk_host_crs_export(self._h, _ptr(rp), None, None, 0))
    self.nnz = int(rp[-1])
    return self


class Dist:
    """spmvtk_dist: one rank of an NCCL communicator (one process per GPU)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * DIST_ID_BYTES)()
        _check(load_library().spmvtk_dist_unique_id(buf))
        return bytes(buf)

    def __init__(self, rank: int, world: int, uid: bytes):
        self._lib = load_library()
        self.rank, self.world = rank, world
        buf = (C.c_ubyte * DIST_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(self._lib.spmvtk_dist_init(rank, world, buf, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def shard(self, config: int, param: int, dparam: float = 0.0, seed: int = 2407) -> "Matrix":
        """This rank's shard of a BASELINE workload (generated shard-only)."""
        return Matrix._make(self._lib.spmvtk_gen_baseline_shard, self._h, config, param,
                            float(dparam), seed)

    def distribute(self, n: int, row_ptr, col_idx, values, index_base: int = 0) -> "Matrix":
        """This rank's shard of a global host CRS (entry-balanced row blocks)."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        return Matrix._make(self._lib.spmvtk_matrix_distribute, self._h, n, _ptr(rp), _ptr(ci),
                            _ptr(v), 8, index_base)

    def iterate(self, shard: "Matrix", kernel: "Kernel", x_ptr: int, steps: int) -> float:
        """x <- A^steps x on the device vector at x_ptr (every rank); returns
        this rank's device seconds per step."""
        sec = C.c_double()
        _check(self._lib.spmvtk_dist_spmv_iterate(self._h, shard.handle, int(kernel),
                                                  C.c_void_p(x_ptr), steps, C.byref(sec)))
        return sec.value

    def push(self, shard: "Matrix", kernel: "Kernel", sparse: bool = True) -> "DistPush":
        """The exchange folded into the SpMV (spmvtk_dist_push_*)."""
        h = C.c_void_p()
        _check(self._lib.spmvtk_dist_push_create(self._h, shard.handle, int(kernel),
                                                 1 if sparse else 0, C.byref(h)))
        return DistPush(self._lib, h, shard)

    def free(self) -> None:
        if self._h:
            self._lib.spmvtk_dist_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass


class DistPush:
    """spmvtk_dist_push: x <- A^steps x with every step one pushed-SpMV launch."""

    def __init__(self, lib, h, shard):
        self._lib, self._h, self._shard = lib, h, shard

    def iterate(self, x_ptr: int, steps: int) -> float:
        sec = C.c_double()
        _check(self._lib.spmvtk_dist_push_iterate(self._h, C.c_void_p(x_ptr), steps,
                                                  C.byref(sec)))
        return sec.value

    def free(self) -> None:
        if self._h:
            self._lib.spmvtk_dist_push_free(self._h)
            self._h = None
