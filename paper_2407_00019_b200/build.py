"""Builds the in-tree native library ``libspmvtk.so`` (sm_100a kernels + host
C++ runtime + C ABI) with the Makefile in ``csrc/``.

nvcc cross-compiles for ``-gencode arch=compute_100a,code=sm_100a`` without a
GPU, so this runs on the CPU build host; the resulting ``.so`` sits next to
this file and travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspmvtk.so")


def build(jobs: int | None = None, verbose: bool = False) -> str:
    jobs = jobs or max(1, min(16, os.cpu_count() or 1))
    cmd = ["make", "-C", CSRC, f"-j{jobs}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stdout.write(res.stdout)
        sys.stderr.write(res.stderr)
    if res.returncode != 0:
        raise RuntimeError("native build failed (see output above)")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
