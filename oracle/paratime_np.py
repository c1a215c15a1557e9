"""ORACLE — numpy restatement of the reference's hot path.  Test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import this module; it is the checker, never the thing measured or shipped.

Every function cites the file:line of ``/root/reference/proj`` it restates.  Where the
reference's operation order is observable in fp64 (the propagator, restriction,
linear interpolation, finite-difference gradients, sums) the numpy expressions keep
that order so results are bitwise equal to the reference compiled without FMA
(``-O3`` and no ``-march``, CMakeLists.txt:3-10).  FFT-based maps (Fourier
interpolation, spectral gradient, the inverse energy map) use ``numpy.fft`` in place
of FFTW; QR/SVD use LAPACK through scipy (dgeqp3/dorgqr, dgesdd) in place of Eigen's
ColPivHouseholderQR / BDCSVD.  Those agree with the reference to round-off.

Layout: fields are numpy arrays shaped ``grid.shape`` (``(n,)`` in 1D, ``(ny, nx)`` in
2D, axis 0 = y), states are ``(u, udot)`` pairs, batches add a leading axis.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import scipy.linalg

FD2, FD4, FD6, FD8, SPECTRAL = 0, 1, 2, 3, 4
SCHEME_NAMES = {"fd2": FD2, "fd4": FD4, "fd6": FD6, "fd8": FD8, "spectral": SPECTRAL}
FOURIER, LINEAR = 0, 1
PLAIN, THETA, CORRECTED_COARSE_ONLY, OMEGA_IDENTITY = 0, 1, 2, 3


class PropagationDiverged(RuntimeError):
    """errors.hpp:9-12"""


# --------------------------------------------------------------------------- grid.hpp


@dataclass(frozen=True)
class Grid:
    """grid.cpp:24-49 — uniform periodic grid, 1 or 2 axes, >= 4 points per axis."""

    n: Tuple[int, ...]
    h: Tuple[float, ...]

    def __post_init__(self):
        if len(self.n) not in (1, 2) or len(self.n) != len(self.h):
            raise ValueError("Grid: dimension must be 1 or 2 with matching spacing")
        for n, h in zip(self.n, self.h):
            if n < 4:
                raise ValueError("Grid: need at least 4 points per axis")
            if not (h > 0.0) or not math.isfinite(h):
                raise ValueError("Grid: spacing must be positive")

    @property
    def dim(self) -> int:
        return len(self.n)

    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(self.n)

    @property
    def size(self) -> int:
        return int(np.prod(self.n))

    def extent(self, axis: int) -> float:
        return float(self.n[axis]) * self.h[axis]

    def cell_volume(self) -> float:
        v = 1.0
        for h in self.h:
            v *= h
        return v


def grid2(ny, nx, hy, hx) -> Grid:
    return Grid((int(ny), int(nx)), (float(hy), float(hx)))


def grid1(n, h) -> Grid:
    return Grid((int(n),), (float(h),))


def finite(u, udot) -> bool:
    """grid.cpp:60"""
    return bool(np.all(np.isfinite(u)) and np.all(np.isfinite(udot)))


@dataclass
class Transfer:
    """grid.cpp:100-119 — nested coarse/fine grids, integer ratio per axis."""

    coarse: Grid
    fine: Grid
    kind: int = FOURIER
    ratio: Tuple[int, ...] = field(init=False)

    def __post_init__(self):
        if self.coarse.dim != self.fine.dim:
            raise ValueError("GridTransfer: dimension mismatch")
        r = []
        for a in range(self.coarse.dim):
            nc, nf = self.coarse.n[a], self.fine.n[a]
            if nf % nc != 0:
                raise ValueError("GridTransfer: fine points must be an integer multiple of coarse points")
            r.append(nf // nc)
            ec, ef = self.coarse.extent(a), self.fine.extent(a)
            if abs(ec - ef) > 1e-12 * max(ec, ef):
                raise ValueError("GridTransfer: coarse and fine extents differ; grids are not nested")
        self.ratio = tuple(r)


def restrict_field(f: np.ndarray, t: Transfer) -> np.ndarray:
    """grid.cpp:121-139 — pointwise: out[j] = in[ratio*j]."""
    if t.coarse.dim == 1:
        return np.ascontiguousarray(f[..., :: t.ratio[0]])
    return np.ascontiguousarray(f[..., :: t.ratio[0], :: t.ratio[1]])


def _signed_freq(k: np.ndarray, n: int) -> np.ndarray:
    """fft.cpp:92-95"""
    return np.where(k <= (n - 1) // 2, k, k - n)


def _fourier_interp_lines(lines: np.ndarray, r: int) -> np.ndarray:
    """grid.cpp:151-177 along the last axis (Nyquist split 1/2-1/2, real part)."""
    if r == 1:
        return lines.copy()
    n = lines.shape[-1]
    m = n * r
    spec = np.fft.fft(lines, axis=-1)
    scale = float(m) / float(n)
    pad = np.zeros(lines.shape[:-1] + (m,), dtype=np.complex128)
    k = np.arange(n)
    nyq = (n % 2 == 0)
    s = _signed_freq(k, n)
    kf = np.where(s >= 0, s, m + s)
    regular = np.ones(n, dtype=bool)
    if nyq:
        regular[n // 2] = False
    pad[..., kf[regular]] = scale * spec[..., regular]
    if nyq:
        half = 0.5 * scale * spec[..., n // 2]
        pad[..., n // 2] += half
        pad[..., m - n // 2] += half
    return np.real(np.fft.ifft(pad, axis=-1))


def _linear_interp_lines(lines: np.ndarray, r: int) -> np.ndarray:
    """grid.cpp:179-191 — out[q*r+rem] = (1-t)*a + t*b, t = rem/r, periodic wrap."""
    if r == 1:
        return lines.copy()
    n = lines.shape[-1]
    a = lines
    b = np.roll(lines, -1, axis=-1)
    out = np.empty(lines.shape[:-1] + (n * r,), dtype=np.float64)
    for rem in range(r):
        t = float(rem) / float(r)
        out[..., rem::r] = (1.0 - t) * a + t * b
    return out


def interpolate_field(f: np.ndarray, t: Transfer) -> np.ndarray:
    """grid.cpp:201-230 — 1D line, or 2D: x within each row, then y within each column."""
    line = _fourier_interp_lines if t.kind == FOURIER else _linear_interp_lines
    if t.coarse.dim == 1:
        return line(f, t.ratio[0])
    half = line(f, t.ratio[1])                                   # along x (axis -1)
    tall = line(np.swapaxes(half, -1, -2), t.ratio[0])           # along y
    return np.ascontiguousarray(np.swapaxes(tall, -1, -2))


# --------------------------------------------------------------------- propagator.cpp


def cfl_check(grid: Grid, c: np.ndarray, dt: float, steps: int) -> None:
    """propagator.cpp:11-27 (PropagatorConfig constructor)."""
    if c.shape != grid.shape:
        raise ValueError("PropagatorConfig: speed field lives on a different grid")
    if not (dt > 0.0) or not math.isfinite(dt):
        raise ValueError("PropagatorConfig: dt must be positive")
    if steps == 0:
        raise ValueError("PropagatorConfig: steps_per_coupling must be positive")
    cmax = float(np.max(c))
    hmin = min(grid.h)
    cfl = dt * cmax / hmin
    bound = 1.0 / math.sqrt(float(grid.dim))
    if cfl > bound * (1.0 + 1e-12):
        raise ValueError("PropagatorConfig: CFL violated")


def laplacian(f: np.ndarray, grid: Grid) -> np.ndarray:
    """propagator.cpp:31-58 — periodic 5-point, x term first, reference operation order."""
    if grid.dim == 1:
        ih2 = 1.0 / (grid.h[0] * grid.h[0])
        return (np.roll(f, -1, -1) - 2.0 * f + np.roll(f, 1, -1)) * ih2
    ihy2 = 1.0 / (grid.h[0] * grid.h[0])
    ihx2 = 1.0 / (grid.h[1] * grid.h[1])
    return ((np.roll(f, -1, -1) - 2.0 * f + np.roll(f, 1, -1)) * ihx2
            + (np.roll(f, -1, -2) - 2.0 * f + np.roll(f, 1, -2)) * ihy2)


def verlet_steps(u: np.ndarray, udot: np.ndarray, c: np.ndarray, grid: Grid, dt: float,
                 steps: int) -> Tuple[np.ndarray, np.ndarray]:
    """propagator.cpp:60-73 repeated `steps` times (no finite check)."""
    u = np.array(u, dtype=np.float64, copy=True)
    udot = np.array(udot, dtype=np.float64, copy=True)
    c2 = c * c
    half_dt2 = 0.5 * dt * dt
    half_dt = 0.5 * dt
    for _ in range(int(steps)):
        a0 = laplacian(u, grid) * c2
        u += dt * udot + half_dt2 * a0
        a1 = laplacian(u, grid)
        udot += half_dt * (a0 + c2 * a1)
    return u, udot


def propagate_coupling(u, udot, c, grid: Grid, dt: float, steps: int):
    """propagator.cpp:95-105 — raises PropagationDiverged on a non-finite result."""
    out = verlet_steps(u, udot, c, grid, dt, steps)
    if not finite(*out):
        raise PropagationDiverged("propagate_coupling: non-finite state produced")
    return out


# --------------------------------------------------------------------- energy_map.cpp

STENCILS = {
    FD2: [1.0 / 2.0],
    FD4: [2.0 / 3.0, -1.0 / 12.0],
    FD6: [3.0 / 4.0, -3.0 / 20.0, 1.0 / 60.0],
    FD8: [4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0],
}  # energy_map.cpp:31-44


def _wavenumbers(grid: Grid, axis: int) -> np.ndarray:
    """fft.cpp:97-100"""
    n = grid.n[axis]
    return 2.0 * math.pi * _signed_freq(np.arange(n), n).astype(np.float64) / grid.extent(axis)


def gradient_axis(f: np.ndarray, grid: Grid, axis: int, scheme: int) -> np.ndarray:
    """energy_map.cpp:50-135 — antisymmetric central differences or FFT derivative."""
    ax = -1 if grid.dim == 1 or axis == 1 else -2
    if scheme == SPECTRAL:
        spec = np.fft.fftn(f, axes=(-2, -1)) if grid.dim == 2 else np.fft.fft(f, axis=-1)
        n = grid.n[axis]
        xi = _wavenumbers(grid, axis)
        mult = 1j * xi
        if n % 2 == 0:
            mult[n // 2] = 0.0  # energy_map.cpp:103-106
        shape = [1] * f.ndim
        shape[ax] = n
        spec = spec * mult.reshape(shape)
        back = np.fft.ifftn(spec, axes=(-2, -1)) if grid.dim == 2 else np.fft.ifft(spec, axis=-1)
        return np.real(back)
    beta = STENCILS[scheme]
    acc = 0.0
    for j, b in enumerate(beta, start=1):
        acc = acc + b * (np.roll(f, -j, ax) - np.roll(f, j, ax))
    return acc * (1.0 / grid.h[axis])


def seq_sum(x: np.ndarray, axis=-1) -> np.ndarray:
    """Left-to-right accumulation (the reference's scalar loops)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[axis] == 0:
        return np.zeros(np.delete(x.shape, axis))
    return np.take(np.add.accumulate(x, axis=axis), -1, axis=axis)


def to_energy_components(u, udot, c, grid: Grid, scheme: int):
    """energy_map.cpp:137-150 — returns (stacked [grad0; grad1; momentum] flat, mean_u)."""
    blocks = [gradient_axis(u, grid, a, scheme) for a in range(grid.dim)]
    momentum = udot / c
    lead = u.shape[: u.ndim - grid.dim]
    flat = [b.reshape(lead + (-1,)) for b in blocks] + [momentum.reshape(lead + (-1,))]
    stacked = np.concatenate(flat, axis=-1)
    mean_u = seq_sum(u.reshape(lead + (-1,)))
    return stacked, mean_u


def from_energy_components(stacked: np.ndarray, mean_u, c: np.ndarray, grid: Grid):
    """energy_map.cpp:152-214 — u_hat = -i (xi.g_hat)/|xi|^2, u_hat(0) = mean_u,
    both-Nyquist bin zeroed; udot = c * momentum."""
    n = grid.size
    d = grid.dim
    blocks = [stacked[..., a * n:(a + 1) * n].reshape(stacked.shape[:-1] + grid.shape) for a in range(d)]
    momentum = stacked[..., d * n:(d + 1) * n].reshape(stacked.shape[:-1] + grid.shape)
    if d == 1:
        xi = _wavenumbers(grid, 0)
        num = xi * np.fft.fft(blocks[0], axis=-1)
        with np.errstate(divide="ignore", invalid="ignore"):
            uhat = (-1j) * num / (xi * xi)
        uhat[..., 0] = mean_u
        u = np.real(np.fft.ifft(uhat, axis=-1))
    else:
        ny, nx = grid.shape
        xiy = _wavenumbers(grid, 0)[:, None]
        xix = _wavenumbers(grid, 1)[None, :]
        num = xiy * np.fft.fftn(blocks[0], axes=(-2, -1)) + xix * np.fft.fftn(blocks[1], axes=(-2, -1))
        with np.errstate(divide="ignore", invalid="ignore"):
            uhat = (-1j) * num / (xiy * xiy + xix * xix)
        uhat[..., 0, 0] = mean_u
        if ny % 2 == 0 and nx % 2 == 0:
            uhat[..., ny // 2, nx // 2] = 0.0
        u = np.real(np.fft.ifftn(uhat, axes=(-2, -1)))
    return u, c * momentum


def energy_of_stacked(stacked: np.ndarray, grid: Grid) -> np.ndarray:
    """energy_map.cpp:216-222 — 0.5 * sum(v*v) * cell volume, sequential sum."""
    return 0.5 * seq_sum(stacked * stacked) * grid.cell_volume()


def energy(u, udot, c, grid: Grid, scheme: int):
    """energy_map.cpp:224-226"""
    return energy_of_stacked(to_energy_components(u, udot, c, grid, scheme)[0], grid)


def energy_error(a, b, c, grid: Grid, scheme: int) -> float:
    """energy_map.cpp:228-236 — sqrt(E(a-b)/E(b)); domain error when E(b)=0."""
    ref = float(energy(b[0], b[1], c, grid, scheme))
    if ref == 0.0:
        raise ZeroDivisionError("energy_error: reference state has zero energy")
    return math.sqrt(float(energy(a[0] - b[0], a[1] - b[1], c, grid, scheme)) / ref)


def l2_error(a_u, b_u) -> float:
    """energy_map.cpp:238-249"""
    d = (a_u - b_u).ravel()
    diff = float(seq_sum(d * d))
    ref = float(seq_sum(b_u.ravel() * b_u.ravel()))
    if ref == 0.0:
        raise ZeroDivisionError("l2_error: reference displacement is zero")
    return math.sqrt(diff / ref)


# ---------------------------------------------------------------------- procrustes.cpp


@dataclass
class Corrector:
    """procrustes.hpp:22-60 — truncated factors X (left), S, Y (right)."""

    X: np.ndarray
    S: np.ndarray
    Y: np.ndarray
    tol: float = 0.0

    @property
    def rows(self) -> int:
        return self.X.shape[0]

    @property
    def rank(self) -> int:
        return self.S.shape[0]

    def empty(self) -> bool:
        return self.X.shape[0] == 0

    def apply(self, v: np.ndarray) -> np.ndarray:
        """procrustes.cpp:82-86 — X (Y^T v)."""
        return self.X @ (self.Y.T @ v)

    def drop_leading(self, count: int) -> "Corrector":
        """procrustes.cpp:88-93"""
        if count < 0:
            raise ValueError("drop_leading: negative count")
        keep = max(0, self.rank - count)
        first = self.rank - keep
        return Corrector(self.X[:, first:].copy(), self.S[first:].copy(), self.Y[:, first:].copy(), self.tol)


def empty_corrector() -> Corrector:
    return Corrector(np.zeros((0, 0)), np.zeros(0), np.zeros((0, 0)))


def _check_tol(tol: float) -> None:
    """procrustes.cpp:14-17"""
    if not (tol > 0.0) or not (tol < 1.0):
        raise ValueError("truncation tolerance must lie in (0, 1)")


def fix_signs(X: np.ndarray, Y: np.ndarray) -> None:
    """procrustes.cpp:21-30 (first maximum on ties)."""
    if X.shape[0] == 0:
        return
    for j in range(X.shape[1]):
        i = int(np.argmax(np.abs(X[:, j])))
        if X[i, j] < 0.0:
            X[:, j] = -X[:, j]
            Y[:, j] = -Y[:, j]


def truncated_qr(A: np.ndarray, drop_tol: float):
    """procrustes.cpp:34-46 — column-pivoted thin QR, R un-pivoted, keep leading
    pivoted |R_ii| > drop_tol."""
    m, n = A.shape
    k = min(m, n)
    if k == 0:
        return np.zeros((m, 0)), np.zeros((0, n))
    Q, R, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
    diag = np.abs(np.diag(R))
    keep = 0
    while keep < k and diag[keep] > drop_tol:
        keep += 1
    Rk = np.zeros((keep, n))
    Rk[:, piv] = np.triu(R[:keep, :])
    return Q[:, :keep].copy(), Rk


def _thin_svd(M: np.ndarray):
    if min(M.shape) == 0:
        k = min(M.shape)
        return np.zeros((M.shape[0], k)), np.zeros(k), np.zeros((M.shape[1], k))
    U, s, Vt = scipy.linalg.svd(M, full_matrices=False, lapack_driver="gesdd")
    return U, s, Vt.T


def _truncate(sigma: np.ndarray, tol: float) -> int:
    smax = sigma[0] if sigma.size else 0.0
    keep = 0
    while keep < sigma.size and smax > 0.0 and sigma[keep] / smax > tol:
        keep += 1
    return keep


def solve_from_scratch(F: np.ndarray, G: np.ndarray, tol: float) -> Corrector:
    """procrustes.cpp:48-69"""
    qr_guard = 1e-14
    QF, RF = truncated_qr(F, qr_guard * np.linalg.norm(F))
    QG, RG = truncated_qr(G, qr_guard * np.linalg.norm(G))
    if QF.shape[1] == 0 or QG.shape[1] == 0:
        return Corrector(np.zeros((F.shape[0], 0)), np.zeros(0), np.zeros((F.shape[0], 0)), tol)
    U, sigma, V = _thin_svd(RF @ RG.T)
    s = _truncate(sigma, tol)
    X = QF @ U[:, :s]
    Y = QG @ V[:, :s]
    fix_signs(X, Y)
    return Corrector(X, sigma[:s].copy(), Y, tol)


def procrustes_solve(F, G, tol) -> Corrector:
    """procrustes.cpp:177-186"""
    _check_tol(tol)
    if F.shape != G.shape:
        raise ValueError("procrustes_solve: F and G must have the same shape")
    if F.shape[1] > F.shape[0]:
        raise ValueError("procrustes_solve: more snapshots than rows")
    if F.shape[1] == 0:
        raise ValueError("procrustes_solve: empty data")
    return solve_from_scratch(F, G, tol)


def update_svd(corr: Corrector, F: np.ndarray, G: np.ndarray, tol: float) -> Corrector:
    """procrustes.cpp:188-237 (Algorithm 1)."""
    _check_tol(tol)
    if F.shape != G.shape:
        raise ValueError("update_svd: F and G must have the same shape")
    if corr.empty():
        return solve_from_scratch(F, G, tol)
    if F.shape[0] != corr.rows:
        raise ValueError("update_svd: block rows do not match corrector")
    U, V, r = corr.X, corr.Y, corr.rank
    UF = U.T @ F
    VG = V.T @ G
    qr_guard = 1e-14
    QF, RF = truncated_qr(F - U @ UF, qr_guard * np.linalg.norm(F))
    QG, RG = truncated_qr(G - V @ VG, qr_guard * np.linalg.norm(G))
    left_block = np.vstack([UF, RF])
    right_block = np.vstack([VG, RG])
    H = left_block @ right_block.T
    H[np.arange(r), np.arange(r)] += corr.S
    Uh, sigma, Vh = _thin_svd(H)
    keep = _truncate(sigma, tol)
    Uext = np.hstack([U, QF])
    Vext = np.hstack([V, QG])
    X = Uext @ Uh[:, :keep]
    Y = Vext @ Vh[:, :keep]
    fix_signs(X, Y)
    return Corrector(X, sigma[:keep].copy(), Y, tol)


def relative_residual(corr: Corrector, F: np.ndarray, G: np.ndarray) -> float:
    """procrustes.cpp:245-253"""
    fnorm = float(np.linalg.norm(F))
    if fnorm == 0.0:
        return 0.0
    if corr.rank == 0:
        return 1.0
    return float(np.linalg.norm(F - corr.X @ (corr.Y.T @ G))) / fnorm


def assemble_snapshots(fine_states, coarse_states, t: Transfer, c_coarse, scheme):
    """procrustes.cpp:158-175 — columns of F, G = stacked components on the coarse grid."""
    if len(fine_states) == 0 or len(fine_states) != len(coarse_states):
        raise ValueError("assemble_snapshots: need equal, nonempty snapshot lists")
    F = np.stack([to_energy_components(restrict_field(s[0], t), restrict_field(s[1], t), c_coarse,
                                       t.coarse, scheme)[0] for s in fine_states], axis=1)
    G = np.stack([to_energy_components(s[0], s[1], c_coarse, t.coarse, scheme)[0]
                  for s in coarse_states], axis=1)
    return F, G


# ------------------------------------------------------------------------ parareal.cpp


@dataclass
class Schedule:
    """parareal.cpp:172-188 (CouplingSchedule) + the two PropagatorConfigs."""

    T: float
    dt_com: float
    n: int
    fine_grid: Grid
    c_fine: np.ndarray
    dt_fine: float
    m_fine: int
    coarse_grid: Grid
    c_coarse: np.ndarray
    dt_coarse: float
    m_coarse: int

    def __post_init__(self):
        cfl_check(self.fine_grid, self.c_fine, self.dt_fine, self.m_fine)
        cfl_check(self.coarse_grid, self.c_coarse, self.dt_coarse, self.m_coarse)
        if not (self.T > 0.0) or not (self.dt_com > 0.0) or self.n == 0:
            raise ValueError("CouplingSchedule: T, dt_com, N must be positive")
        if abs(float(self.n) * self.dt_com - self.T) > 1e-9 * self.T:
            raise ValueError("CouplingSchedule: N * dt_com must equal T")
        for m, dt in ((self.m_fine, self.dt_fine), (self.m_coarse, self.dt_coarse)):
            if abs(float(m) * dt - self.dt_com) > 1e-12 * self.dt_com:
                raise ValueError("CouplingSchedule: steps_per_coupling * dt != dt_com")


@dataclass
class Record:
    """parareal.hpp:29-37"""

    states: List[Tuple[np.ndarray, np.ndarray]]
    energy_err: np.ndarray
    l2_err: np.ndarray
    residual: float = float("nan")
    rank: int = 0
    diverged: bool = False


@dataclass
class Run:
    reference: List[Tuple[np.ndarray, np.ndarray]]
    iterations: List[Record]


def _nan_state(grid: Grid):
    """parareal.cpp:49-54"""
    return np.full(grid.shape, np.nan), np.full(grid.shape, np.nan)


def fine_stage(s, sch: Schedule):
    """parareal.cpp:58-64"""
    try:
        return propagate_coupling(s[0], s[1], sch.c_fine, sch.fine_grid, sch.dt_fine, sch.m_fine)
    except PropagationDiverged:
        return _nan_state(sch.fine_grid)


def coarse_stage(s, sch: Schedule, t: Transfer):
    """parareal.cpp:66-73"""
    try:
        return propagate_coupling(restrict_field(s[0], t), restrict_field(s[1], t), sch.c_coarse,
                                  sch.coarse_grid, sch.dt_coarse, sch.m_coarse)
    except PropagationDiverged:
        return _nan_state(t.coarse)


def _measure(state, ref, c, grid, scheme):
    """parareal.cpp:80-103"""
    inf = float("inf")
    if not finite(*state) or not finite(*ref):
        return inf, inf
    ref_energy = float(energy(ref[0], ref[1], c, grid, scheme))
    if ref_energy == 0.0:
        e = 0.0 if float(energy(state[0] - ref[0], state[1] - ref[1], c, grid, scheme)) == 0.0 else inf
    else:
        e = energy_error(state, ref, c, grid, scheme)
    ref_l2 = float(seq_sum(ref[0].ravel() * ref[0].ravel()))
    if ref_l2 == 0.0:
        d = (state[0] - ref[0]).ravel()
        l2 = 0.0 if float(seq_sum(d * d)) == 0.0 else inf
    else:
        l2 = l2_error(state[0], ref[0])
    return e, l2


def _finalize(states, previous, reference, sch: Schedule, metric_scheme: int, keep_states=True) -> Record:
    """parareal.cpp:107-128 — errors vs reference, flag and clamp non-finite states."""
    count = len(states)
    ee = np.zeros(count)
    l2 = np.zeros(count)
    diverged = False
    for n in range(count):
        if n == 0:
            e = (0.0, 0.0)
        else:
            e = _measure(states[n], reference[n], sch.c_fine, sch.fine_grid, metric_scheme)
        ee[n], l2[n] = e
        if not finite(*states[n]):
            diverged = True
            if previous is not None:
                states[n] = previous[n]
    return Record(states=list(states) if keep_states else [], energy_err=ee, l2_err=l2, diverged=diverged)


def serial_fine(init, sch: Schedule):
    """parareal.cpp:190-199 (raises PropagationDiverged)."""
    states = [init]
    for _ in range(sch.n):
        states.append(propagate_coupling(states[-1][0], states[-1][1], sch.c_fine, sch.fine_grid,
                                         sch.dt_fine, sch.m_fine))
    return states


def _reference_or_nan(init, sch: Schedule):
    """parareal.cpp:133-145"""
    try:
        return serial_fine(init, sch)
    except PropagationDiverged:
        return [init] + [_nan_state(sch.fine_grid) for _ in range(sch.n)]


def _interp_state(s, t):
    return interpolate_field(s[0], t), interpolate_field(s[1], t)


def _serial_coarse_init(init, sch, t):
    """parareal.cpp:147-159"""
    states = [init]
    for _ in range(sch.n):
        co = coarse_stage(states[-1], sch, t)
        states.append(_interp_state(co, t) if finite(*co) else _nan_state(t.fine))
    return states


def _validate(init, sch, t, iterations):
    """parareal.cpp:161-168"""
    if init[0].shape != sch.fine_grid.shape:
        raise ValueError("parareal: initial state must live on the fine grid")
    if t.fine != sch.fine_grid or t.coarse != sch.coarse_grid:
        raise ValueError("parareal: transfer does not couple the schedule grids")
    if iterations < 0:
        raise ValueError("parareal: negative iteration count")


def plain_parareal(init, sch: Schedule, t: Transfer, iterations: int, metric_scheme=FD2,
                   keep_states=True) -> Run:
    """parareal.cpp:201-237 — next = I C R next[n-1] + F cur[n-1] - I C R cur[n-1]."""
    _validate(init, sch, t, iterations)
    N = sch.n
    reference = _reference_or_nan(init, sch)
    current = _serial_coarse_init(init, sch, t)
    run = Run(reference=reference, iterations=[_finalize(current, None, reference, sch, metric_scheme, keep_states)])
    for _ in range(iterations):
        fine_next = [None] + [fine_stage(current[n - 1], sch) for n in range(1, N + 1)]
        coarse_next = [None]
        for n in range(1, N + 1):
            co = coarse_stage(current[n - 1], sch, t)
            coarse_next.append(_interp_state(co, t) if finite(*co) else _nan_state(t.fine))
        nxt = [init]
        for n in range(1, N + 1):
            cn = coarse_stage(nxt[n - 1], sch, t)
            cnf = _interp_state(cn, t) if finite(*cn) else _nan_state(t.fine)
            nxt.append(((cnf[0] + fine_next[n][0]) - coarse_next[n][0],
                        (cnf[1] + fine_next[n][1]) - coarse_next[n][1]))
        run.iterations.append(_finalize(nxt, current, reference, sch, metric_scheme, keep_states))
        current = nxt
    return run


def _corrected_coarse_state(s, corr: Corrector, c_coarse, grid, scheme, omega_identity):
    """parareal.cpp:245-253 — Lambda, Omega (or identity), Lambda-dagger."""
    stacked, mean_u = to_energy_components(s[0], s[1], c_coarse, grid, scheme)
    if not omega_identity:
        stacked = corr.apply(stacked)
    return from_energy_components(stacked, mean_u, c_coarse, grid)


def theta_parareal(init, sch: Schedule, t: Transfer, iterations: int, scheme=FD2, tol=1e-15,
                   omega_identity=False, additive_correction=True, remove_leading=0,
                   metric_scheme=FD2, keep_states=True) -> Run:
    """parareal.cpp:255-350 (theta_engine; Algorithm 3)."""
    _validate(init, sch, t, iterations)
    N = sch.n
    c_coarse = sch.c_coarse
    reference = _reference_or_nan(init, sch)
    current = _serial_coarse_init(init, sch, t)
    run = Run(reference=reference, iterations=[_finalize(current, None, reference, sch, metric_scheme, keep_states)])
    corrector = empty_corrector()
    for _ in range(iterations):
        fine_next = [None] + [fine_stage(current[n - 1], sch) for n in range(1, N + 1)]
        coarse_next = [None] + [coarse_stage(current[n - 1], sch, t) for n in range(1, N + 1)]
        keep = [n for n in range(1, N + 1) if finite(*fine_next[n]) and finite(*coarse_next[n])]
        residual, rank = float("nan"), 0
        applied = corrector
        if keep:
            F, G = assemble_snapshots([fine_next[n] for n in keep], [coarse_next[n] for n in keep], t,
                                      c_coarse, scheme)
            if omega_identity:
                fn = float(np.linalg.norm(F))
                residual = float(np.linalg.norm(F - G)) / fn if fn > 0.0 else 0.0
            else:
                corrector = update_svd(corrector, F, G, tol)
                applied = corrector.drop_leading(remove_leading) if remove_leading > 0 else corrector
                residual = relative_residual(applied, F, G)
                rank = applied.rank
        elif not omega_identity:
            applied = corrector.drop_leading(remove_leading)
            rank = applied.rank
        nxt = [init]
        for n in range(1, N + 1):
            if additive_correction:
                if n == 1:
                    nxt.append(fine_next[1])
                    continue
                w = coarse_stage(nxt[n - 1], sch, t)
                if not finite(*w) or not finite(*coarse_next[n]) or not finite(*fine_next[n]):
                    nxt.append(_nan_state(t.fine))
                    continue
                cnew = _corrected_coarse_state(w, applied, c_coarse, t.coarse, scheme, omega_identity)
                cold = _corrected_coarse_state(coarse_next[n], applied, c_coarse, t.coarse, scheme,
                                               omega_identity)
                d = _interp_state((cnew[0] - cold[0], cnew[1] - cold[1]), t)
                nxt.append((fine_next[n][0] + d[0], fine_next[n][1] + d[1]))
            else:
                w = coarse_stage(nxt[n - 1], sch, t)
                if not finite(*w):
                    nxt.append(_nan_state(t.fine))
                    continue
                nxt.append(_interp_state(_corrected_coarse_state(w, applied, c_coarse, t.coarse, scheme,
                                                                 omega_identity), t))
        rec = _finalize(nxt, current, reference, sch, metric_scheme, keep_states)
        rec.residual, rec.rank = residual, rank
        run.iterations.append(rec)
        current = nxt
    return run


def corrected_coarse_only(init, sch, t, iterations, **kw) -> Run:
    """parareal.cpp:359-365"""
    kw["additive_correction"] = False
    return theta_parareal(init, sch, t, iterations, **kw)
