"""paratime_b200 — B200-native hot path of data-driven theta-parareal (arXiv 1905.00473).

The product is ``libparatime_b200.so`` (CUDA kernels for sm_100a + the extern "C"
ABI of ``include/paratime_b200.h`` + the C++ drop-in of ``include/paratime/*.hpp``).
This Python package is plumbing: it loads the library with ctypes and hands it
device pointers of torch tensors.  There is no CPU fallback — if the library or a
CUDA device is missing, every entry point raises.
"""
from __future__ import annotations

from .api import (  # noqa: F401
    DIVERGED,
    EXACT,
    FAST,
    FD2,
    FD4,
    FD6,
    FD8,
    FOURIER,
    LINEAR,
    SPECTRAL,
    Context,
    Grid,
    PtbError,
    PmlPropagator,
    Propagator,
    damping_profile,
    pml_parareal_run,
    pml_theta_run,
    Transfer,
    lib,
    lib_path,
)
