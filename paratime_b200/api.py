"""ctypes binding of libparatime_b200.so (include/paratime_b200.h).

Device memory is owned by torch tensors (plumbing); the library only sees raw
pointers.  The context runs on torch's current CUDA stream so library kernels and
torch ops are stream-ordered.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence, Tuple

import numpy as np

LIB = Path(__file__).resolve().parent / "libparatime_b200.so"

OK, INVALID_ARGUMENT, DIVERGED, DOMAIN, CUDA_ERR, NCCL_ERR, UNSUPPORTED, CONFIG = range(8)
FAST, EXACT = 0, 1
FOURIER, LINEAR = 0, 1
FD2, FD4, FD6, FD8, SPECTRAL = range(5)

_lib = None


class PtbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[ptb status {status}] {msg}")
        self.status = status


class _Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_size_t * 2), ("h", C.c_double * 2)]


def lib_path() -> Path:
    # PTB_LIB: an alternate build of the same library (A/B measurements of kernel variants only)
    return Path(os.environ["PTB_LIB"]) if os.environ.get("PTB_LIB") else LIB


def lib():
    """Load the CUDA library; raises (no fallback) when it has not been built."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not path.exists():
            raise ImportError(f"{path} is missing — build it with `python -m paratime_b200.build`")
        _lib = C.CDLL(str(path))
        _lib.ptb_last_error.restype = C.c_char_p
        _lib.ptb_version.restype = C.c_char_p
        _lib.ptb_context_stream.restype = C.c_void_p
        _lib.ptb_context_launches.restype = C.c_uint64
        _lib.ptb_propagator_speed.restype = C.c_void_p
    return _lib


def check(status: int) -> None:
    if status != OK:
        raise PtbError(status, lib().ptb_last_error().decode())


@dataclass(frozen=True)
class Grid:
    """grid.hpp:16-38 — n/h per axis, axis 0 = y in 2D."""

    n: Tuple[int, ...]
    h: Tuple[float, ...]

    @property
    def dim(self) -> int:
        return len(self.n)

    @property
    def shape(self):
        return tuple(self.n)

    @property
    def size(self) -> int:
        return int(np.prod(self.n))

    def c(self) -> _Grid:
        g = _Grid()
        g.dim = self.dim
        g.n[0], g.n[1] = self.n[0], (self.n[1] if self.dim == 2 else 1)
        g.h[0], g.h[1] = self.h[0], (self.h[1] if self.dim == 2 else 1.0)
        return g

    @staticmethod
    def of(g) -> "Grid":
        return Grid(tuple(int(x) for x in g.n), tuple(float(x) for x in g.h))


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(None)


class Context:
    """ptb_context: device + stream + scratch.  Follows torch's current stream."""

    def __init__(self, device: int = 0):
        import torch

        self.torch = torch
        self.device = device
        h = C.c_void_p()
        check(lib().ptb_context_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.follow_torch_stream()

    def follow_torch_stream(self):
        s = self.torch.cuda.current_stream(self.device).cuda_stream
        check(lib().ptb_context_set_stream(self.h, C.c_void_p(s)))

    def use_own_stream(self):
        """Issue this context's work on its own stream instead of torch's current one (in-process
        loopback ranks: each rank's work stays in its own stream, as in one-process-per-GPU runs)."""
        check(lib().ptb_context_use_own_stream(self.h))
        return self

    def launches(self) -> int:
        return int(lib().ptb_context_launches(self.h))

    def synchronize(self):
        check(lib().ptb_context_synchronize(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().ptb_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # helpers
    def tensor(self, a, dtype=None):
        t = self.torch.as_tensor(np.ascontiguousarray(a), dtype=dtype or self.torch.float64)
        return t.to(f"cuda:{self.device}")

    def laplacian(self, grid: Grid, f):
        batch = f.numel() // grid.size
        out = self.torch.empty_like(f)
        check(lib().ptb_laplacian_batch(self.h, C.byref(grid.c()), C.c_size_t(batch), _ptr(f), _ptr(out)))
        return out

    def nonfinite(self, f, n: int):
        batch = f.numel() // n
        flags = self.torch.zeros(batch, dtype=self.torch.int32, device=f.device)
        check(lib().ptb_nonfinite_batch(self.h, C.c_size_t(n), C.c_size_t(batch), _ptr(f), _ptr(flags)))
        return flags


class Propagator:
    """PropagatorConfig (propagator.hpp:12-21) living on the device."""

    def __init__(self, ctx: Context, grid: Grid, c, dt: float, steps: int):
        self.ctx, self.grid, self.dt, self.steps = ctx, grid, float(dt), int(steps)
        c = np.ascontiguousarray(c, dtype=np.float64).reshape(-1)
        if c.size != grid.size:
            raise PtbError(INVALID_ARGUMENT, "SpeedField: field size does not match grid")
        h = C.c_void_p()
        check(lib().ptb_propagator_create(ctx.h, C.byref(grid.c()), c.ctypes.data_as(C.POINTER(C.c_double)),
                                          C.c_double(dt), C.c_size_t(steps), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ptb_propagator_destroy(self.h)
        except Exception:
            pass

    def propagate(self, u, udot, mode: int = FAST, steps: Optional[int] = None, flags=None):
        """In place on device tensors (batch, *grid.shape) or grid.shape."""
        batch = u.numel() // self.grid.size
        if steps is None:
            check(lib().ptb_propagate_batch(self.h, C.c_size_t(batch), _ptr(u), _ptr(udot), _ptr(flags), C.c_int(mode)))
        else:
            check(lib().ptb_propagate_steps_batch(self.h, C.c_size_t(steps), C.c_size_t(batch), _ptr(u), _ptr(udot),
                                                  _ptr(flags), C.c_int(mode)))
        return u, udot

    def plan(self, batch: int, mode: int = FAST, steps: Optional[int] = None) -> str:
        """Launch plan propagate() would use (kernel names, strip widths, grids)."""
        buf = C.create_string_buffer(512)
        nsteps = self.steps if steps is None else steps
        check(lib().ptb_propagate_plan(self.h, C.c_size_t(nsteps), C.c_size_t(batch), C.c_int(mode), buf,
                                       C.c_size_t(len(buf))))
        return buf.value.decode()

    def propagate_host(self, u: np.ndarray, udot: np.ndarray, mode: int = FAST):
        """propagate_coupling on host arrays; raises PtbError(DIVERGED) like the reference."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        udot = np.ascontiguousarray(udot, dtype=np.float64)
        uo, vo = np.empty_like(u), np.empty_like(udot)
        dp = C.POINTER(C.c_double)
        check(lib().ptb_propagate_coupling_host(self.h, u.ctypes.data_as(dp), udot.ctypes.data_as(dp),
                                                uo.ctypes.data_as(dp), vo.ctypes.data_as(dp), C.c_int(mode)))
        return uo, vo


class PmlPropagator:
    """Absorbing-layer fine propagator (config 4; not in the reference, scheme in oracle/pml_np.py).

    State: u, udot, px, py device tensors of shape (batch, ny, nx) or (ny, nx); px, py zero
    outside the layer.  zeta_y / zeta_x: damping per row / column (damping_profile)."""

    def __init__(self, ctx: Context, grid: Grid, c, zeta_y, zeta_x, dt: float, steps: int):
        self.ctx, self.grid, self.dt, self.steps = ctx, grid, float(dt), int(steps)
        dp = C.POINTER(C.c_double)
        c = np.ascontiguousarray(c, dtype=np.float64).reshape(-1)
        zy = np.ascontiguousarray(zeta_y, dtype=np.float64).reshape(-1)
        zx = np.ascontiguousarray(zeta_x, dtype=np.float64).reshape(-1)
        if c.size != grid.size or grid.dim != 2 or zy.size != grid.n[0] or zx.size != grid.n[1]:
            raise PtbError(INVALID_ARGUMENT, "PmlConfig: field sizes do not match the 2D grid")
        h = C.c_void_p()
        check(lib().ptb_pml_create(ctx.h, C.byref(grid.c()), c.ctypes.data_as(dp), zy.ctypes.data_as(dp),
                                   zx.ctypes.data_as(dp), C.c_double(dt), C.c_size_t(steps), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ptb_pml_destroy(self.h)
        except Exception:
            pass

    def propagate(self, u, udot, px, py, steps: Optional[int] = None, flags=None):
        import torch

        n = self.grid.size
        batch = u.numel() // n
        dev = torch.device("cuda", self.ctx.device)
        for name, t in (("u", u), ("udot", udot), ("px", px), ("py", py)):
            if (t.dtype != torch.float64 or not t.is_contiguous() or t.device != dev
                    or t.numel() != batch * n or batch == 0):
                raise PtbError(INVALID_ARGUMENT, f"pml propagate: {name} must be a contiguous float64 tensor of "
                               f"batch x {n} values on {dev}")
        if flags is not None and (flags.dtype != torch.int32 or flags.numel() < batch or flags.device != dev):
            raise PtbError(INVALID_ARGUMENT, "pml propagate: flags must be int32[batch] on the context's device")
        check(lib().ptb_pml_propagate_batch(self.h, C.c_size_t(steps or 0), C.c_size_t(batch), _ptr(u), _ptr(udot),
                                            _ptr(px), _ptr(py), _ptr(flags)))
        return u, udot, px, py


def pml_parareal_run(fine: "PmlPropagator", coarse: "PmlPropagator", transfer: "Transfer", n_couplings: int,
                     iterations: int, u0, udot0, keep_states: bool = False, comm: "Comm" = None):
    """ptb_pml_parareal_run: plain parareal with the absorbing layer.  Returns a dict with the
    L2 distances to the serial fine run relative to the initial state [K x (N+1)], per-iteration device ms, the diverged flag and (optionally)
    the last iterate as an array [4, N+1, *grid] (u, udot, px, py)."""
    N, K = int(n_couplings), int(iterations)
    dp = C.POINTER(C.c_double)
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    v0 = np.ascontiguousarray(udot0, dtype=np.float64)
    if u0.size != fine.grid.size or v0.size != fine.grid.size:
        raise PtbError(INVALID_ARGUMENT, "pml_parareal_run: initial state does not match the fine grid")
    err = np.zeros((max(K, 1), N + 1))
    ms = np.zeros(max(K, 1))
    states = np.empty((4, N + 1) + tuple(fine.grid.n)) if keep_states else None
    div = C.c_int32(0)
    out = (err.ctypes.data_as(dp), ms.ctypes.data_as(dp), states.ctypes.data_as(dp) if keep_states else None,
           C.byref(div))
    if comm is None:
        check(lib().ptb_pml_parareal_run(fine.h, coarse.h, transfer.h, C.c_size_t(N), C.c_int(K),
                                         u0.ctypes.data_as(dp), v0.ctypes.data_as(dp), *out))
    else:  # slices sharded over the ranks of `comm`; states filled for the own slices only
        check(lib().ptb_pml_parareal_run_sharded(fine.h, coarse.h, transfer.h, comm.h, C.c_size_t(N), C.c_int(K),
                                                 u0.ctypes.data_as(dp), v0.ctypes.data_as(dp), *out))
    return {"rel_err": err[:K], "iteration_ms": ms[:K], "diverged": bool(div.value), "states": states}


def pml_theta_run(fine: "PmlPropagator", coarse: "PmlPropagator", transfer: "Transfer", n_couplings: int,
                  iterations: int, u0, udot0, tol: float = 1e-4, scheme: int = 0, keep_states: bool = False,
                  comm: "Comm" = None):
    """ptb_pml_theta_run: theta (Procrustes) parareal with the absorbing layer (oracle/pml_np.py
    theta_parareal).  Returns pml_parareal_run's dict plus per-iteration corrector "rank" and "residual"."""
    N, K = int(n_couplings), int(iterations)
    dp = C.POINTER(C.c_double)
    n_f = int(np.prod(fine.grid.n))
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    v0 = np.ascontiguousarray(udot0, dtype=np.float64)
    if u0.size != n_f or v0.size != n_f:
        raise PtbError(INVALID_ARGUMENT, "pml_theta_run: initial state does not match the fine grid")
    err = np.zeros((max(K, 1), N + 1))
    ms = np.zeros(max(K, 1))
    ranks = np.zeros(max(K, 1), dtype=np.int32)
    res = np.zeros(max(K, 1))
    states = np.empty((4, N + 1) + tuple(fine.grid.n)) if keep_states else None
    div = C.c_int32(0)
    check(lib().ptb_pml_theta_run(fine.h, coarse.h, transfer.h, comm.h if comm is not None else None,
                                  C.c_size_t(N), C.c_int(K), C.c_double(tol), C.c_int(scheme),
                                  u0.ctypes.data_as(dp), v0.ctypes.data_as(dp), err.ctypes.data_as(dp),
                                  ms.ctypes.data_as(dp), states.ctypes.data_as(dp) if keep_states else None,
                                  ranks.ctypes.data_as(C.POINTER(C.c_int32)), res.ctypes.data_as(dp), C.byref(div)))
    return {"rel_err": err[:K], "iteration_ms": ms[:K], "diverged": bool(div.value), "states": states,
            "rank": ranks[:K], "residual": res[:K]}


def damping_profile(n: int, width: int, h: float, cmax: float, reflection: float = 1e-4) -> np.ndarray:
    """ptb_pml_damping_profile (host): quadratic profile on `width` cells at both ends."""
    out = np.empty(n)
    check(lib().ptb_pml_damping_profile(C.c_size_t(n), C.c_size_t(width), C.c_double(h), C.c_double(cmax),
                                        C.c_double(reflection), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


class Transfer:
    """GridTransfer (grid.hpp:56-67): restriction and interpolation on the device."""

    def __init__(self, ctx: Context, coarse: Grid, fine: Grid, kind: int = FOURIER):
        self.ctx, self.coarse, self.fine, self.kind = ctx, coarse, fine, kind
        h = C.c_void_p()
        check(lib().ptb_transfer_create(ctx.h, C.byref(coarse.c()), C.byref(fine.c()), C.c_int(kind), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ptb_transfer_destroy(self.h)
        except Exception:
            pass

    def restrict(self, f):
        batch = f.numel() // self.fine.size
        out = self.ctx.torch.empty((batch,) + self.coarse.shape, dtype=f.dtype, device=f.device)
        check(lib().ptb_restrict_batch(self.h, C.c_size_t(batch), _ptr(f), _ptr(out)))
        return out

    def interpolate(self, f):
        batch = f.numel() // self.coarse.size
        out = self.ctx.torch.empty((batch,) + self.fine.shape, dtype=f.dtype, device=f.device)
        check(lib().ptb_interpolate_batch(self.h, C.c_size_t(batch), _ptr(f), _ptr(out)))
        return out


# ---------------------------------------------------------------- energy map / DFT


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def write_speed_model(grid: Grid, c) -> str:
    """Speed-model text (experiment.hpp:90): "ny nx dy dx" header, ny rows of nx values (%.17g)."""
    c = np.ascontiguousarray(c, dtype=np.float64).ravel()
    need = C.c_size_t()
    check(lib().ptb_speed_model_write(C.byref(grid.c()), _dp(c), None, C.c_size_t(0), C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(lib().ptb_speed_model_write(C.byref(grid.c()), _dp(c), buf, C.c_size_t(need.value), C.byref(need)))
    return buf.value.decode()


def run_csv(energy_err, l2_err, residual, rank, diverged, plain: bool, which: str) -> str:
    """The reference harness's run-record CSV text (experiment.cpp:596-628): which is "errors",
    "residuals" or "summary"; energy_err / l2_err are K x (N + 1), the rest length K."""
    ee = np.ascontiguousarray(energy_err, dtype=np.float64)
    l2 = np.ascontiguousarray(l2_err, dtype=np.float64)
    res = np.ascontiguousarray(residual, dtype=np.float64)
    rk = np.ascontiguousarray(rank, dtype=np.int32)
    dv = np.ascontiguousarray(diverged, dtype=np.int32)
    K, N1 = ee.shape
    w = {"errors": 0, "residuals": 1, "summary": 2}[which]
    args = (C.c_size_t(K), C.c_size_t(N1), _dp(ee), _dp(l2), _dp(res), rk.ctypes.data_as(C.c_void_p),
            dv.ctypes.data_as(C.c_void_p), C.c_int(int(plain)), C.c_int(w))
    need = C.c_size_t()
    check(lib().ptb_run_csv(*args, None, C.c_size_t(0), C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(lib().ptb_run_csv(*args, buf, C.c_size_t(need.value), C.byref(need)))
    return buf.value.decode()


def read_speed_model(text: str):
    """read_speed_model (experiment.hpp:86): (Grid, c as grid.shape); PtbError(CONFIG) on malformed
    input, as the reference's ConfigError."""
    g = _Grid()
    npts = C.c_size_t()
    raw = text.encode()
    check(lib().ptb_speed_model_read(raw, C.byref(g), None, C.c_size_t(0), C.byref(npts)))
    c = np.empty(npts.value)
    check(lib().ptb_speed_model_read(raw, C.byref(g), _dp(c), C.c_size_t(npts.value), C.byref(npts)))
    grid = Grid((int(g.n[0]),), (float(g.h[0]),)) if g.dim == 1 else Grid((int(g.n[0]), int(g.n[1])),
                                                                           (float(g.h[0]), float(g.h[1])))
    return grid, c.reshape(grid.shape)


def energy_components(ctx: Context, grid: Grid, c_dev, scheme: int, u, udot):
    """Lambda on `batch` device states -> (stacked (batch, (d+1)N), mean (batch,))."""
    batch = u.numel() // grid.size
    rows = (grid.dim + 1) * grid.size
    out = ctx.torch.empty((batch, rows), dtype=ctx.torch.float64, device=u.device)
    mean = ctx.torch.empty(batch, dtype=ctx.torch.float64, device=u.device)
    check(lib().ptb_energy_components_batch(ctx.h, C.byref(grid.c()), _ptr(c_dev), C.c_int(scheme), C.c_size_t(batch),
                                            _ptr(u), _ptr(udot), _ptr(out), C.c_size_t(rows), _ptr(mean)))
    return out, mean


def from_energy_components(ctx: Context, grid: Grid, c_dev, stacked, mean):
    batch = stacked.shape[0]
    rows = (grid.dim + 1) * grid.size
    u = ctx.torch.empty((batch,) + grid.shape, dtype=ctx.torch.float64, device=stacked.device)
    v = ctx.torch.empty_like(u)
    check(lib().ptb_from_energy_components_batch(ctx.h, C.byref(grid.c()), _ptr(c_dev), C.c_size_t(batch),
                                                 _ptr(stacked), C.c_size_t(rows), _ptr(mean), _ptr(u), _ptr(v)))
    return u, v


def energy_sums(ctx: Context, grid: Grid, c_dev, scheme: int, ua, va, ub, vb):
    batch = ua.numel() // grid.size
    out = ctx.torch.empty((batch, 4), dtype=ctx.torch.float64, device=ua.device)
    check(lib().ptb_energy_sums_batch(ctx.h, C.byref(grid.c()), _ptr(c_dev), C.c_int(scheme), C.c_size_t(batch),
                                      _ptr(ua), _ptr(va), _ptr(ub), _ptr(vb), _ptr(out)))
    return out


def dft(ctx: Context, grid: Grid, data_complex, inverse=False):
    """In-place DFT of a complex128 device tensor (batch, *grid.shape)."""
    batch = data_complex.numel() // grid.size
    check(lib().ptb_dft_batch(ctx.h, C.byref(grid.c()), C.c_size_t(batch), _ptr(data_complex), C.c_int(int(inverse))))
    return data_complex


# ---------------------------------------------------------------- Procrustes corrector


class Corrector:
    """PhaseCorrector (procrustes.hpp:22-60) with device-resident factors."""

    def __init__(self, ctx: Context, handle=None):
        self.ctx = ctx
        if handle is None:
            handle = C.c_void_p()
            check(lib().ptb_corrector_create(ctx.h, C.byref(handle)))
        self.h = handle

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ptb_corrector_destroy(self.h)
        except Exception:
            pass

    def update(self, F, G, tol: float):
        """update_svd in place; F, G: device (cols, rows) tensors = column-major rows x cols."""
        if tuple(F.shape) != tuple(G.shape):
            raise PtbError(INVALID_ARGUMENT, "update_svd: F and G must have the same shape")
        cols, rows = F.shape
        check(lib().ptb_corrector_update(self.h, C.c_size_t(rows), C.c_size_t(cols), _ptr(F), _ptr(G), C.c_double(tol)))
        return self

    def solve(self, F, G, tol: float):
        if tuple(F.shape) != tuple(G.shape):
            raise PtbError(INVALID_ARGUMENT, "procrustes_solve: F and G must have the same shape")
        cols, rows = F.shape
        check(lib().ptb_procrustes_solve(self.h, C.c_size_t(rows), C.c_size_t(cols), _ptr(F), _ptr(G), C.c_double(tol)))
        return self

    def shape(self):
        r, k = C.c_size_t(), C.c_size_t()
        check(lib().ptb_corrector_shape(self.h, C.byref(r), C.byref(k)))
        return r.value, k.value

    def factors(self):
        rows, rank = self.shape()
        X = np.empty((rank, rows))
        Y = np.empty((rank, rows))
        S = np.empty(rank)
        check(lib().ptb_corrector_factors(self.h, _dp(X), _dp(S), _dp(Y)))
        return X.T.copy(), S, Y.T.copy()

    def drop_leading(self, count: int) -> "Corrector":
        out = C.c_void_p()
        check(lib().ptb_corrector_drop_leading(self.h, C.c_size_t(count), C.byref(out)))
        return Corrector(self.ctx, out)

    def apply(self, V):
        """V: device (batch, rows) -> X (Y^T v) per row vector."""
        out = self.ctx.torch.empty_like(V)
        check(lib().ptb_corrector_apply_batch(self.h, C.c_size_t(V.shape[0]), _ptr(V), _ptr(out)))
        return out

    def residual(self, F, G) -> float:
        cols, rows = F.shape
        out = C.c_double()
        check(lib().ptb_relative_residual(self.h, C.c_size_t(rows), C.c_size_t(cols), _ptr(F), _ptr(G), C.byref(out)))
        return out.value


# ---------------------------------------------------------------- drivers

PLAIN, THETA, CORRECTED_COARSE_ONLY, OMEGA_IDENTITY = range(4)
MAX_TIMED = 64


class RunSpec(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("fine_n", C.c_size_t * 2), ("fine_h", C.c_double * 2), ("coarse_n", C.c_size_t * 2),
        ("coarse_h", C.c_double * 2), ("dt_fine", C.c_double), ("m_fine", C.c_size_t), ("dt_coarse", C.c_double),
        ("m_coarse", C.c_size_t), ("T", C.c_double), ("dt_com", C.c_double), ("n_couplings", C.c_size_t),
        ("interp", C.c_int), ("iterations", C.c_int), ("variant", C.c_int), ("scheme", C.c_int),
        ("metric_scheme", C.c_int), ("tol", C.c_double), ("remove_leading", C.c_int), ("mode", C.c_int),
    ]


class PhaseTimes(C.Structure):
    _fields_ = [("reference_ms", C.c_double), ("gather_ms", C.c_double * MAX_TIMED),
                ("parallel_ms", C.c_double * MAX_TIMED),
                ("procrustes_ms", C.c_double * MAX_TIMED), ("sweep_ms", C.c_double * MAX_TIMED),
                ("finalize_ms", C.c_double * MAX_TIMED), ("iteration_ms", C.c_double * MAX_TIMED)]


def run_spec(**kw) -> RunSpec:
    s = RunSpec()
    for k, v in kw.items():
        if k in ("fine_n", "coarse_n", "fine_h", "coarse_h"):
            arr = getattr(s, k)
            arr[0] = v[0]
            arr[1] = v[1] if len(v) > 1 else (1 if "n" in k else 1.0)
        else:
            setattr(s, k, v)
    return s


class Comm:
    """NCCL communicator for slice sharding (one process per GPU).  `broadcast` sends rank 0's
    128-byte unique id to every rank (e.g. via torch.distributed)."""

    def __init__(self, ctx: Context, rank: int, world: int, broadcast=None):
        self.rank, self.world = rank, world
        uid = C.create_string_buffer(128)
        if world > 1:
            if rank == 0:
                check(lib().ptb_nccl_unique_id(uid))
            raw = broadcast(bytes(uid.raw)) if broadcast else bytes(uid.raw)
            uid = C.create_string_buffer(raw, 128)
        h = C.c_void_p()
        check(lib().ptb_comm_create(ctx.h, C.c_int(rank), C.c_int(world), uid, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ptb_comm_destroy(self.h)
        except Exception:
            pass


class LoopbackGroup:
    """In-process ranks for the sharded driver (one thread per rank)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib().ptb_loopback_group_create(C.c_int(world), C.byref(h)))
        self.h, self.world = h, world

    def comm(self, ctx: Context, rank: int) -> "Comm":
        c = Comm.__new__(Comm)
        c.rank, c.world = rank, self.world
        h = C.c_void_p()
        check(lib().ptb_comm_create_loopback(ctx.h, self.h, C.c_int(rank), C.byref(h)))
        c.h = h
        return c

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ptb_loopback_group_destroy(self.h)
        except Exception:
            pass


def parareal_run(ctx: Context, spec: RunSpec, c_fine, c_coarse, u0, udot0, keep_states=False,
                 keep_reference=False, comm: "Comm" = None):
    """plain / theta / corrected-coarse-only parareal on the device (parareal.cpp); with `comm`
    the slices are sharded over the ranks (states then hold this rank's slices only)."""
    K, N = spec.iterations, spec.n_couplings
    fine_shape = (spec.fine_n[0],) if spec.dim == 1 else (spec.fine_n[0], spec.fine_n[1])
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    cf, cc, u0, v0 = f(c_fine), f(c_coarse), f(u0), f(udot0)
    ee = np.empty((K + 1, N + 1))
    l2 = np.empty((K + 1, N + 1))
    res = np.empty(K + 1)
    rank = np.empty(K + 1, dtype=np.int32)
    div = np.empty(K + 1, dtype=np.int32)
    states = np.empty((K + 1, N + 1, 2) + fine_shape) if keep_states else None
    ref = np.empty((N + 1, 2) + fine_shape) if keep_reference else None
    times = PhaseTimes()
    ip = C.POINTER(C.c_int)
    check(lib().ptb_parareal_run_sharded(ctx.h, comm.h if comm is not None else None, C.byref(spec), _dp(cf), _dp(cc),
                                         _dp(u0), _dp(v0), _dp(ee), _dp(l2), _dp(res), rank.ctypes.data_as(ip),
                                         div.ctypes.data_as(ip), _dp(states) if states is not None else None,
                                         _dp(ref) if ref is not None else None, C.byref(times)))
    k = min(K, MAX_TIMED)
    t = {"reference_ms": times.reference_ms}
    for name in ("parallel_ms", "gather_ms", "procrustes_ms", "sweep_ms", "finalize_ms", "iteration_ms"):
        t[name] = list(getattr(times, name))[:k]
    return dict(energy_err=ee, l2_err=l2, residual=res, rank=rank, diverged=div, states=states, reference=ref,
                times=t)
