"""B200-native run-time sparse transformation + SpMV + auto-tuning path of
arXiv 2407.00019 (reference: "spmvtk").

The product is the native library ``libspmvtk.so`` built from ``csrc/``
(sm_100a CUDA kernels, host C++ runtime, the reference's C ABI); ``spmvtk``
is its Python binding and ``dist`` the row-block multi-GPU driver.
"""
from . import spmvtk  # noqa: F401
from .spmvtk import (Array, Decision, Format, Kernel, Matrix, Profile,  # noqa: F401
                     SpmvtkError, Status, load_library)

__all__ = ["spmvtk", "Array", "Decision", "Format", "Kernel", "Matrix", "Profile",
           "SpmvtkError", "Status", "load_library"]
