"""CPU oracle (test infrastructure only) for the absorbing-layer fine propagator of config 4.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module.

PARITY UNPINNED.  The reference has no absorbing layer: its propagator is periodic only
(propagator.cpp:31-105; SPEC.md:8,97 names a PML as future work) and SURVEY.md 8(f) rank 4 states
that BASELINE.json config 4's "32-cell perfectly-matched absorbing layer" has no oracle.  This file
is the specification of the scheme the CUDA kernel implements (csrc/pml.cu); it is pinned by
self-consistency instead of by the reference:
  * with a zero damping profile the step is the periodic fine propagator (oracle/paratime_np.py
    verlet_steps, i.e. propagator.cpp:60-73) to round-off, and the GPU kernel equals the periodic
    FAST kernel bitwise;
  * a pulse that leaves the interior is absorbed (reflection well below the interior signal of a
    boundary-free reference run on a larger periodic box);
  * energy in the interior decays once the wave has entered the layer and stays bounded (stable).

Continuous model (Grote & Sim's auxiliary-field PML for the second-order wave equation, written
for the non-divergence operator c^2 Lap u of the reference):
    u_tt + (zx + zy) u_t + zx zy u = c^2 (Lap u + d/dx px + d/dy py)
    px_t = -zx px + (zy - zx) du/dx,     py_t = -zy py + (zx - zy) du/dy
zx(x), zy(y) >= 0 vanish in the interior, so there px = py = 0 and the equation is u_tt = c^2 Lap u.

Discrete step (dt, hd = dt/2, Kx = hd c^2 / hx^2 as the FAST kernel; D = centred difference):
    F(u, p)  = Kx (cc u + ry (uN + uS) + (uW + uE)) + Kx (gx (pxE - pxW) + gy (pyN - pyS)),
               gx = hx / 2, gy = hx^2 / (2 hy)          [= hd c^2 (Lap u + Dx px + Dy py)]
    vh  = v + (F(u, p) - hd (pi u + sg v))               sg = zx + zy, pi = zx zy
    u1  = u + dt vh
    px1 = ax px + bx (u1E - u1W)     ax = (1 - hd zx)/(1 + hd zx), bx = (zy - zx) qx,
                                     qx = dt / (2 hx (1 + hd zx))          (py likewise)
    v1  = (vh + (F(u1, p1) - hd pi u1)) * inv            inv = 1 / (1 + hd sg)
i.e. velocity Verlet with the damping split trapezoidally over the two half kicks and the auxiliary
fields advanced by the trapezoidal (Crank-Nicolson) rule for their decay.  With zx = zy = 0 the
step is kick-drift-kick Verlet, the periodic propagator.
"""
from __future__ import annotations

import numpy as np


def damping_profile(n: int, width: int, h: float, cmax: float, reflection: float = 1e-4) -> np.ndarray:
    """Quadratic profile zeta(d) = z0 (d/L)^2 on the first and last `width` cells of a periodic axis.

    d is the distance of the cell centre into the layer (cells width-1-i+1/2 ... 1/2 from the
    interior edge), L = width*h, z0 = (3/2) cmax ln(1/R) / L (the standard quadratic-profile
    amplitude for a theoretical normal-incidence reflection R).  Computed with plain IEEE
    operations in this order by both the oracle and the C++ host code (csrc/pml.cu ptb_pml_damping_profile).
    """
    z = np.zeros(n)
    if width <= 0:
        return z
    if 2 * width >= n:
        raise ValueError("pml: layer wider than half the axis")
    L = width * h
    z0 = 1.5 * cmax * np.log(1.0 / reflection) / L
    for i in range(width):
        t = (width - i - 0.5) / width
        z[i] = z0 * (t * t)
        z[n - 1 - i] = z0 * (t * t)
    return z


class PmlCoefficients:
    """Host-computed coefficients (the same expressions as csrc/pml.cu's pml_create)."""

    def __init__(self, c: np.ndarray, hy: float, hx: float, dt: float, zy: np.ndarray, zx: np.ndarray):
        ny, nx = c.shape
        assert zy.shape == (ny,) and zx.shape == (nx,)
        self.dt = dt
        self.hd = 0.5 * dt
        ihx2 = 1.0 / (hx * hx)
        ihy2 = 1.0 / (hy * hy)
        self.ry = ihy2 / ihx2
        self.cc = -2.0 * (1.0 + self.ry)
        self.kx = self.hd * (c * c) * ihx2
        self.gx = 0.5 * hx
        self.gy = (hx * hx) / (2.0 * hy)
        self.zx = zx.astype(np.float64)
        self.zy = zy.astype(np.float64)
        self.ax = (1.0 - self.hd * zx) / (1.0 + self.hd * zx)
        self.ay = (1.0 - self.hd * zy) / (1.0 + self.hd * zy)
        self.qx = dt / (2.0 * hx * (1.0 + self.hd * zx))
        self.qy = dt / (2.0 * hy * (1.0 + self.hd * zy))
        sg = zy[:, None] + zx[None, :]
        self.sg = sg
        self.pi = zy[:, None] * zx[None, :]
        self.inv = 1.0 / (1.0 + self.hd * sg)
        self.bx = (zy[:, None] - zx[None, :]) * self.qx[None, :]
        self.by = (zx[None, :] - zy[:, None]) * self.qy[:, None]


def _sh(f, dy, dx):
    """f at (iy + dy, ix + dx), periodic."""
    return np.roll(f, (-dy, -dx), axis=(-2, -1))


def _force(u, px, py, k: PmlCoefficients):
    b = k.kx * ((k.cc * u + k.ry * (_sh(u, 1, 0) + _sh(u, -1, 0))) + (_sh(u, 0, -1) + _sh(u, 0, 1)))
    div = k.kx * (k.gx * (_sh(px, 0, 1) - _sh(px, 0, -1)) + k.gy * (_sh(py, 1, 0) - _sh(py, -1, 0)))
    return b + div


def pml_steps(u, v, px, py, k: PmlCoefficients, steps: int):
    """`steps` PML Verlet steps of a state (arrays (..., ny, nx)); returns new arrays."""
    u, v, px, py = (np.array(a, dtype=np.float64, copy=True) for a in (u, v, px, py))
    for _ in range(steps):
        vh = v + (_force(u, px, py, k) - k.hd * (k.pi * u + k.sg * v))
        u = u + k.dt * vh
        px = k.ax[None, :] * px + k.bx * (_sh(u, 0, 1) - _sh(u, 0, -1))
        py = k.ay[:, None] * py + k.by * (_sh(u, 1, 0) - _sh(u, -1, 0))
        v = (vh + (_force(u, px, py, k) - k.hd * (k.pi * u))) * k.inv
    return u, v, px, py


def interior_energy(u, v, c, hy, hx, width: int):
    """0.5 sum (|grad u|^2 + (v/c)^2) dx dy over the interior (cells outside the layer), forward
    differences; a diagnostic for the absorption tests, not a reference metric."""
    gx = (_sh(u, 0, 1) - u) / hx
    gy = (_sh(u, 1, 0) - u) / hy
    e = 0.5 * (gx * gx + gy * gy + (v / c) ** 2) * hx * hy
    w = width
    return float(np.sum(e[..., w:e.shape[-2] - w, w:e.shape[-1] - w]))


def plain_parareal(u0, v0, kf: PmlCoefficients, m_f: int, kc: PmlCoefficients, m_c: int, t, N: int, K: int):
    """Plain parareal (Eq. 2; parareal.cpp:201-237) on the layered state (u, udot, px, py), the
    way csrc/pml.cu pml_parareal evaluates it: interpolated px, py are zeroed on undamped cells,
    non-finite iterates are clamped to the previous one; iterate 0 = the interpolated serial coarse chain;
    per iteration fine_next[n] = F(cur[n-1]), old[n] = C(R cur[n-1]); coarse sweep
    w_0 = R(init), d_n = C(w_{n-1}) - old[n], w_n = R(fine_next[n]) + d_n; next[n] = fine_next[n] + I(d_n).
    `t` is an oracle/paratime_np.Transfer.  Returns (iterates per k as lists of 4-tuples,
    L2 distances of [u; udot] to the serial fine run relative to the initial state's norm [K x (N+1)])."""
    from oracle import paratime_np as P

    R = lambda s: tuple(P.restrict_field(f, t) for f in s)  # noqa: E731
    # px, py vanish identically on undamped cells (zx = zy = 0), so their interpolants are cut
    # back to the layer (Fourier I would otherwise spread them over the interior)
    damped = (kf.zy[:, None] != 0.0) | (kf.zx[None, :] != 0.0)

    def I(s):  # noqa: E743
        u, v, px, py = (P.interpolate_field(f, t) for f in s)
        return u, v, np.where(damped, px, 0.0), np.where(damped, py, 0.0)

    def finite(s):
        return all(np.all(np.isfinite(f)) for f in s)

    Fp = lambda s: pml_steps(*s, kf, m_f)  # noqa: E731
    Cp = lambda s: pml_steps(*s, kc, m_c)  # noqa: E731
    z = np.zeros_like(u0)
    init = (u0, v0, z, z)
    ref = [init]
    for _ in range(N):
        ref.append(Fp(ref[-1]))
    cur = [init]
    w = R(init)
    for _ in range(N):
        w = Cp(w)
        cur.append(I(w))
    out, errs = [], []
    for _ in range(K):
        fine_next = [None] + [Fp(cur[n - 1]) for n in range(1, N + 1)]
        old = [None] + [Cp(R(cur[n - 1])) for n in range(1, N + 1)]
        nxt = [init]
        w = R(init)
        for n in range(1, N + 1):
            g = Cp(w)
            d = tuple(a - b for a, b in zip(g, old[n]))
            w = tuple(a + b for a, b in zip(R(fine_next[n]), d))
            nxt.append(tuple(a + b for a, b in zip(fine_next[n], I(d))))
        for n in range(1, N + 1):  # finalize_iteration (parareal.cpp:117-124): clamp non-finite
            if not finite(nxt[n]):
                nxt[n] = cur[n]
        e = []
        den = np.sum(ref[0][0] ** 2 + ref[0][1] ** 2)  # the initial state's norm (the layer drains energy)
        for n in range(N + 1):
            num = np.sum((nxt[n][0] - ref[n][0]) ** 2 + (nxt[n][1] - ref[n][1]) ** 2)
            e.append(float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num)))
        errs.append(e)
        out.append(nxt)
        cur = nxt
    return out, np.array(errs)


def theta_parareal(u0, v0, kf: PmlCoefficients, m_f: int, kc: PmlCoefficients, m_c: int, t, N: int, K: int,
                   c_coarse, tol: float = 1e-4, scheme: int = 0, aux: str = "none"):
    """Theta-parareal (the data-driven Procrustes coupling, parareal.cpp:255-350) on the layered
    state (u, udot, px, py) — this build's extension, the way csrc/pml.cu pml_parareal(theta)
    evaluates it.  The reference defines the coupling on (u, udot) only (energy_map.cpp:137-214);
    with the layer:
      * snapshots F = Lambda(R fine_next[n]), G = Lambda(C(R cur[n-1])) of the (u, udot) part over
        slices whose four fields are finite; corrector = update_svd(corrector, F, G, tol);
      * the sweep corrects (u, udot) with Lambda-dagger Omega Lambda (corrected_coarse_state,
        parareal.cpp:245-253); the auxiliary fields (px, py) are not corrected (aux="none", the
        default: next[n]'s are fine_next[n]'s):
        d = (corr(w) - corr(old[n]))_{u,udot} ++ (0, 0),  w = C(w_{n-1});
        aux="plain" corrects them additively as plain parareal, d_p = (w - old[n])_p — measured
        unstable (scripts/pml_theta_explore.py: the iterates grow from iteration ~5 while the
        corrector rank collapses, as plain parareal does on the whole state);
        n = 1 takes fine_next[1] (both terms cancel exactly, as in parareal.cpp:315-318);
        w_n = R(fine_next[n]) + d (as the plain sweep), next[n] = fine_next[n] + I(d) with the
        auxiliary part masked to the layer; a non-finite w, old[n] or fine_next[n] gives a NaN
        state (parareal.cpp:323-326);
      * finalize: non-finite iterates clamped to the previous one.
    Returns (iterates per k, L2 distances of [u; udot] to the serial fine run relative to the
    initial state's norm [K x (N+1)], corrector ranks per k)."""
    from oracle import paratime_np as P

    R = lambda s: tuple(P.restrict_field(f, t) for f in s)  # noqa: E731
    damped = (kf.zy[:, None] != 0.0) | (kf.zx[None, :] != 0.0)

    def I(s):  # noqa: E743
        u, v, px, py = (P.interpolate_field(f, t) for f in s)
        return u, v, np.where(damped, px, 0.0), np.where(damped, py, 0.0)

    def finite(s):
        return all(np.all(np.isfinite(f)) for f in s)

    Fp = lambda s: pml_steps(*s, kf, m_f)  # noqa: E731
    Cp = lambda s: pml_steps(*s, kc, m_c)  # noqa: E731
    z = np.zeros_like(u0)
    init = (u0, v0, z, z)
    ref = [init]
    for _ in range(N):
        ref.append(Fp(ref[-1]))
    cur = [init]
    w = R(init)
    for _ in range(N):
        w = Cp(w)
        cur.append(I(w))
    corr = P.empty_corrector()
    nan = np.full_like(u0, np.nan)
    out, errs, ranks = [], [], []
    den = np.sum(init[0] ** 2 + init[1] ** 2)
    for _ in range(K):
        fine_next = [None] + [Fp(cur[n - 1]) for n in range(1, N + 1)]
        old = [None] + [Cp(R(cur[n - 1])) for n in range(1, N + 1)]
        keep = [n for n in range(1, N + 1) if finite(fine_next[n]) and finite(old[n])]
        if keep:
            F, G = P.assemble_snapshots([fine_next[n][:2] for n in keep], [old[n][:2] for n in keep], t,
                                        c_coarse, scheme)
            corr = P.update_svd(corr, F, G, tol)
        ranks.append(corr.rank)

        def corrected(s):
            return P._corrected_coarse_state(s[:2], corr, c_coarse, t.coarse, scheme, False)

        nxt = [init]
        w = R(init)
        for n in range(1, N + 1):
            g = Cp(w)
            if n == 1:
                d = tuple(np.zeros_like(f) for f in g)
            elif not (finite(g) and finite(old[n]) and finite(fine_next[n])):
                d = tuple(np.full_like(f, np.nan) for f in g)
            else:
                cn, co = corrected(g), corrected(old[n])
                if aux == "plain":
                    d = (cn[0] - co[0], cn[1] - co[1], g[2] - old[n][2], g[3] - old[n][3])
                else:  # "none": the auxiliary fields take fine_next's as they are
                    d = (cn[0] - co[0], cn[1] - co[1], np.zeros_like(g[2]), np.zeros_like(g[3]))
            w = tuple(a + b for a, b in zip(R(fine_next[n]), d))
            if n == 1:
                nxt.append(fine_next[1])
            elif not np.all(np.isfinite(d[0])):
                nxt.append((nan, nan, nan, nan))
            else:
                nxt.append(tuple(a + b for a, b in zip(fine_next[n], I(d))))
        for n in range(1, N + 1):
            if not finite(nxt[n]):
                nxt[n] = cur[n]
        e = []
        for n in range(N + 1):
            num = np.sum((nxt[n][0] - ref[n][0]) ** 2 + (nxt[n][1] - ref[n][1]) ** 2)
            e.append(float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num)))
        errs.append(e)
        out.append(nxt)
        cur = nxt
    return out, np.array(errs), ranks
