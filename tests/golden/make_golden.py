"""Generates tests/golden/ref_random.npz by running the REFERENCE library
(oracle/_ref/libspmvtk_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile) on small seeded inputs.  Run here, where /root/reference
exists; the fixture travels with the repository so GPU-box tests can pin
parity without the reference sources.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_random.npz")


def main() -> None:
    O.build(ref=True)
    ref = O.Ref()
    rng = np.random.default_rng(20240700019)
    data: dict[str, np.ndarray] = {}
    cases = []
    # random matrices with unsorted columns (test_support.hpp:43-74 shape)
    for _ in range(24):
        cases.append(O.random_crs(rng, 60, 400))
    # edge cases: all rows empty, a single entry, empty leading/trailing rows
    cases.append((4, np.array([1, 1, 1, 1, 1]), np.array([], np.int64), np.array([])))
    cases.append((1, np.array([1, 2]), np.array([1]), np.array([2.5])))
    cases.append((6, np.array([1, 1, 1, 3, 3, 3, 3]), np.array([5, 2]), np.array([1.5, -2.0])))
    for i, (n, rp, ci, v) in enumerate(cases):
        h = ref.matrix(n, rp, ci, v)
        x = rng.uniform(-1.0, 1.0, size=n)
        p = f"m{i}_"
        data[p + "n"] = np.array([n])
        data[p + "row_ptr"] = np.asarray(rp, np.int64)
        data[p + "col_idx"] = np.asarray(ci, np.int64)
        data[p + "values"] = np.asarray(v, np.float64)
        data[p + "x"] = x
        for fmt, name in ((1, "ccs"), (2, "coo_row"), (3, "coo_col"), (4, "ell")):
            rc, out, msg = ref.convert(h, fmt)
            assert rc == 0, msg
            if name == "ccs":
                data[p + "ccs_col_ptr"] = ref.array(out, 1)
                data[p + "ccs_row_idx"] = ref.array(out, 2)
                data[p + "ccs_values"] = ref.array(out, 0)
            elif name.startswith("coo"):
                data[p + name + "_row_idx"] = ref.array(out, 2)
                data[p + name + "_col_idx"] = ref.array(out, 3)
                data[p + name + "_values"] = ref.array(out, 0)
            else:
                meta = ref.meta(out)
                data[p + "ell_band_count"] = np.array([meta["band_count"]])
                data[p + "ell_values"] = ref.array(out, 0)
                data[p + "ell_col_idx"] = ref.array(out, 3)
                data[p + "ell_row_entry_count"] = ref.array(out, 4)
            kernels = {"ccs": [], "coo_row": [1], "coo_col": [2], "ell": [3, 4]}[name]
            for k in kernels:
                for lanes in (1, 3):
                    y, _ = ref.spmv(out, k, x, lanes)
                    data[p + f"y_k{k}_l{lanes}"] = y
            ref.free(out)
        y, _ = ref.spmv(h, 0, x, 1)
        data[p + "y_k0_l1"] = y
        ref.free(h)
    data["count"] = np.array([len(cases)])
    # reference generators (ingest.cpp:234-316) for byte-identity checks
    gens = {
        "banded_200_1": ("banded", 200, 1),
        "banded_300_4": ("banded", 300, 4),
        "skewed_500_2_10_250_99": ("skewed", 500, 2, 10, 250, 99),
        "skewed_10000_1_1_5000_0": ("skewed", 10000, 1, 1, 5000, 0),
        "cv_2000_8_1.5_7": ("cv_target", 2000, 8.0, 1.5, 7),
        "cv_1000_5_0_3": ("cv_target", 1000, 5.0, 0.0, 3),
    }
    for key, (kind, *args) in gens.items():
        h = ref.gen(kind, *args)
        data[f"gen_{key}_row_ptr"] = ref.array(h, 1)
        data[f"gen_{key}_col_idx"] = ref.array(h, 3)
        data[f"gen_{key}_values"] = ref.array(h, 0)
        ref.free(h)
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT}: {len(cases)} matrices, {len(gens)} generator outputs")


if __name__ == "__main__":
    main()
