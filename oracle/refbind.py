"""ORACLE — ctypes binding of oracle/_ref/libparatime_ref.so.  Test infrastructure only.

The library is the reference's own C++ (grid.cpp, propagator.cpp, energy_map.cpp,
parareal.cpp, experiment.cpp compiled verbatim from /root/reference by
``oracle/ref/Makefile``) plus the oracle's restatements of fft.cpp and
procrustes.cpp.  It is built in this container by ``__graft_entry__.build()`` and
shipped to the GPU box as a prebuilt file (``/root/reference`` does not exist there).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional

import numpy as np

from .paratime_np import Grid

LIB_PATH = Path(__file__).resolve().parent / "_ref" / "libparatime_ref.so"
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_sz = C.c_size_t


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class RunSpec(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("fine_n", _sz * 2),
        ("fine_h", C.c_double * 2),
        ("coarse_n", _sz * 2),
        ("coarse_h", C.c_double * 2),
        ("dt_fine", C.c_double),
        ("m_fine", _sz),
        ("dt_coarse", C.c_double),
        ("m_coarse", _sz),
        ("T", C.c_double),
        ("dt_com", C.c_double),
        ("n_couplings", _sz),
        ("interp", C.c_int),
        ("iterations", C.c_int),
        ("variant", C.c_int),
        ("scheme", C.c_int),
        ("metric_scheme", C.c_int),
        ("tol", C.c_double),
        ("remove_leading", C.c_int),
        ("workers", C.c_int),
    ]


REFERENCE_SRC = Path("/root/reference/proj/src")


def build() -> bool:
    """Compile oracle/_ref from the reference sources (only where /root/reference exists)."""
    if not REFERENCE_SRC.exists():
        return LIB_PATH.exists()
    import subprocess

    subprocess.run(["make", "-s", "-C", str(Path(__file__).resolve().parent / "ref"), "-j8"], check=True)
    return LIB_PATH.exists()


def available() -> bool:
    return LIB_PATH.exists() or REFERENCE_SRC.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} not built (run __graft_entry__.build())")
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _check(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _g(grid: Grid):
    if grid.dim == 1:
        return (C.c_int(1), _sz(grid.n[0]), _sz(1), C.c_double(grid.h[0]), C.c_double(1.0))
    return (C.c_int(2), _sz(grid.n[0]), _sz(grid.n[1]), C.c_double(grid.h[0]), C.c_double(grid.h[1]))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def laplacian(f, grid):
    f = _f64(f)
    out = np.empty_like(f)
    _check(lib().ref_laplacian(*_g(grid), _p(f), _p(out)))
    return out


def cfl_check(grid, c, dt, steps):
    c = _f64(c)
    _check(lib().ref_cfl_check(*_g(grid), _p(c), C.c_double(dt), _sz(steps)))


def propagate(u, udot, c, grid, dt, steps, workers=1):
    """Batched propagate_coupling; u, udot shaped (B,)+grid.shape or grid.shape.
    Returns (u, udot, diverged[B])."""
    u = np.array(u, dtype=np.float64, copy=True, order="C")
    udot = np.array(udot, dtype=np.float64, copy=True, order="C")
    c = _f64(c)
    batch = u.size // grid.size
    div = np.zeros(batch, dtype=np.int32)
    _check(lib().ref_propagate(*_g(grid), _p(c), C.c_double(dt), _sz(steps), _sz(batch), _p(u), _p(udot),
                               C.c_int(workers), div.ctypes.data_as(_ip)))
    return u, udot, div


def step(u, udot, c, grid, dt):
    u = np.array(u, dtype=np.float64, copy=True)
    udot = np.array(udot, dtype=np.float64, copy=True)
    c = _f64(c)
    _check(lib().ref_step(*_g(grid), _p(c), C.c_double(dt), _p(u), _p(udot)))
    return u, udot


def _tg(coarse, fine):
    cg, fg = _g(coarse), _g(fine)
    return (cg[0], cg[1], cg[2], cg[3], cg[4], fg[1], fg[2], fg[3], fg[4])


def restrict(f, coarse, fine):
    f = _f64(f)
    out = np.empty(coarse.shape)
    _check(lib().ref_restrict(*_tg(coarse, fine), _p(f), _p(out)))
    return out


def interpolate(f, coarse, fine, kind):
    f = _f64(f)
    out = np.empty(fine.shape)
    _check(lib().ref_interpolate(*_tg(coarse, fine), C.c_int(kind), _p(f), _p(out)))
    return out


def gradient_axis(f, grid, axis, scheme):
    f = _f64(f)
    out = np.empty_like(f)
    _check(lib().ref_gradient_axis(*_g(grid), _p(f), C.c_int(axis), C.c_int(scheme), _p(out)))
    return out


def energy_components(u, udot, c, grid, scheme):
    u, udot, c = _f64(u), _f64(udot), _f64(c)
    out = np.empty((grid.dim + 1) * grid.size)
    mean = C.c_double()
    _check(lib().ref_energy_components(*_g(grid), _p(c), C.c_int(scheme), _p(u), _p(udot), _p(out),
                                       C.byref(mean)))
    return out, mean.value


def from_energy_components(stacked, mean_u, c, grid):
    stacked, c = _f64(stacked), _f64(c)
    u = np.empty(grid.shape)
    udot = np.empty(grid.shape)
    _check(lib().ref_from_energy_components(*_g(grid), _p(c), _p(stacked), C.c_double(mean_u), _p(u), _p(udot)))
    return u, udot


def energy(u, udot, c, grid, scheme):
    u, udot, c = _f64(u), _f64(udot), _f64(c)
    out = C.c_double()
    _check(lib().ref_energy(*_g(grid), _p(c), C.c_int(scheme), _p(u), _p(udot), C.byref(out)))
    return out.value


def energy_error(a, b, c, grid, scheme):
    ua, udota, ub, udotb, c = map(_f64, (a[0], a[1], b[0], b[1], c))
    out = C.c_double()
    _check(lib().ref_energy_error(*_g(grid), _p(c), C.c_int(scheme), _p(ua), _p(udota), _p(ub), _p(udotb),
                                  C.byref(out)))
    return out.value


def l2_error(ua, ub, grid):
    ua, ub = _f64(ua), _f64(ub)
    out = C.c_double()
    _check(lib().ref_l2_error(*_g(grid), _p(ua), _p(ub), C.byref(out)))
    return out.value


class RefCorrector:
    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if self.h and _lib is not None:
            _lib.ref_corrector_free(self.h)
            self.h = None

    def shape(self):
        rows, rank = C.c_long(), C.c_long()
        _check(lib().ref_corrector_shape(self.h, C.byref(rows), C.byref(rank)))
        return rows.value, rank.value

    def factors(self):
        rows, rank = self.shape()
        X = np.empty((rank, rows))
        Y = np.empty((rank, rows))
        S = np.empty(rank)
        _check(lib().ref_corrector_factors(self.h, _p(X), _p(S), _p(Y)))
        return X.T.copy(), S, Y.T.copy()

    def apply(self, v):
        v = _f64(v)
        out = np.empty_like(v)
        _check(lib().ref_corrector_apply(self.h, _p(v), _p(out)))
        return out

    def drop_leading(self, count):
        out = C.c_void_p()
        _check(lib().ref_corrector_drop_leading(self.h, C.c_long(count), C.byref(out)))
        return RefCorrector(out.value)

    def residual(self, F, G):
        F, G = np.asfortranarray(F, dtype=np.float64), np.asfortranarray(G, dtype=np.float64)
        out = C.c_double()
        _check(lib().ref_relative_residual(self.h, C.c_long(F.shape[0]), C.c_long(F.shape[1]), _p(F), _p(G),
                                           C.byref(out)))
        return out.value


def procrustes_solve(F, G, tol):
    F, G = np.asfortranarray(F, dtype=np.float64), np.asfortranarray(G, dtype=np.float64)
    out = C.c_void_p()
    _check(lib().ref_procrustes_solve(C.c_long(F.shape[0]), C.c_long(F.shape[1]), _p(F), _p(G),
                                      C.c_double(tol), C.byref(out)))
    return RefCorrector(out.value)


def update_svd(corr: Optional[RefCorrector], F, G, tol):
    F, G = np.asfortranarray(F, dtype=np.float64), np.asfortranarray(G, dtype=np.float64)
    out = C.c_void_p()
    _check(lib().ref_update_svd(corr.h if corr is not None else None, C.c_long(F.shape[0]),
                                C.c_long(F.shape[1]), _p(F), _p(G), C.c_double(tol), C.byref(out)))
    return RefCorrector(out.value)


def build_setup(preset: str = "", config_text: str = "", overrides: str = ""):
    """Resolve a reference preset/config (experiment.cpp:503-557) into (spec, c_f, c_c, u0, udot0)."""
    spec = RunSpec()
    args = (preset.encode(), config_text.encode(), overrides.encode())
    _check(lib().ref_build_setup(*args, C.byref(spec), None, None, None, None))
    fine = spec_grid(spec, fine=True)
    coarse = spec_grid(spec, fine=False)
    cf, cc = np.empty(fine.shape), np.empty(coarse.shape)
    u0, ud0 = np.empty(fine.shape), np.empty(fine.shape)
    _check(lib().ref_build_setup(*args, C.byref(spec), _p(cf), _p(cc), _p(u0), _p(ud0)))
    return spec, cf, cc, u0, ud0


def spec_grid(spec: RunSpec, fine: bool) -> Grid:
    n = spec.fine_n if fine else spec.coarse_n
    h = spec.fine_h if fine else spec.coarse_h
    if spec.dim == 1:
        return Grid((int(n[0]),), (float(h[0]),))
    return Grid((int(n[0]), int(n[1])), (float(h[0]), float(h[1])))


def parareal_run(spec: RunSpec, c_fine, c_coarse, u0, udot0, keep_states=False, keep_reference=False):
    """The reference's plain_parareal / theta_parareal / corrected_coarse_only (parareal.cpp)."""
    K, N = spec.iterations, spec.n_couplings
    fine = spec_grid(spec, True)
    nf = fine.size
    ee = np.empty((K + 1, N + 1))
    l2 = np.empty((K + 1, N + 1))
    res = np.empty(K + 1)
    rank = np.empty(K + 1, dtype=np.int32)
    div = np.empty(K + 1, dtype=np.int32)
    states = np.empty((K + 1, N + 1, 2) + fine.shape) if keep_states else None
    ref = np.empty((N + 1, 2) + fine.shape) if keep_reference else None
    wall = C.c_double()
    cf, cc, u0, udot0 = map(_f64, (c_fine, c_coarse, u0, udot0))
    _check(lib().ref_parareal_run(C.byref(spec), _p(cf), _p(cc), _p(u0), _p(udot0), _p(ee), _p(l2), _p(res),
                                  rank.ctypes.data_as(_ip), div.ctypes.data_as(_ip),
                                  _p(states) if states is not None else None,
                                  _p(ref) if ref is not None else None, C.byref(wall)))
    return dict(energy_err=ee, l2_err=l2, residual=res, rank=rank, diverged=div, states=states,
                reference=ref, wall_ms=wall.value)

