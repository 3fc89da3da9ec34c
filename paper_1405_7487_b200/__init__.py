"""B200-native (sm_100a) 3D Laplace FMM hot path of arXiv 1405.7487 behind a C-ABI.

`FMM(n_max, P, theta, ncrit, prec)` wraps libfmm.so (include/fmm.h); see DESIGN.md.
"""
from .fmm import FMM, FMMError, lib, LIB_PATH, SYMBOLS  # noqa: F401

__all__ = ["FMM", "FMMError", "lib", "LIB_PATH", "SYMBOLS"]
