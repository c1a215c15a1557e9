"""Implementations under test, behind one small interface.

``OracleImpl`` is the numpy restatement (oracle/paratime_np.py) — the CPU checker.
``CudaImpl`` drives the B200 library through its C ABI (paratime_b200, ctypes).
The known-answer checks in tests/kat.py run against both, so a GPU test reads like
the reference's own doctest case it restates.
"""
from __future__ import annotations

import numpy as np

from oracle import paratime_np as P


class Diverged(Exception):
    pass


class InvalidArgument(Exception):
    pass


class OracleImpl:
    name = "oracle"

    def grid(self, n, h):
        try:
            return P.Grid(tuple(int(x) for x in n), tuple(float(x) for x in h))
        except ValueError as e:
            raise InvalidArgument(str(e))

    def laplacian(self, f, grid):
        return P.laplacian(np.asarray(f, dtype=np.float64), grid)

    def check_config(self, grid, c, dt, steps):
        try:
            P.cfl_check(grid, np.asarray(c, dtype=np.float64).reshape(grid.shape), dt, steps)
        except ValueError as e:
            raise InvalidArgument(str(e))

    def propagate(self, u, udot, c, grid, dt, steps):
        self.check_config(grid, c, dt, steps)
        try:
            return P.propagate_coupling(np.asarray(u, float).reshape(grid.shape), np.asarray(udot, float).reshape(grid.shape),
                                        np.asarray(c, float).reshape(grid.shape), grid, dt, steps)
        except P.PropagationDiverged as e:
            raise Diverged(str(e))

    def propagate_batch(self, u, udot, c, grid, dt, steps):
        return P.verlet_steps(u, udot, np.asarray(c, float).reshape(grid.shape), grid, dt, steps)

    def transfer(self, coarse, fine, kind):
        try:
            return P.Transfer(coarse, fine, kind)
        except ValueError as e:
            raise InvalidArgument(str(e))

    def restrict(self, f, t):
        return P.restrict_field(np.asarray(f, float), t)

    def interpolate(self, f, t):
        return P.interpolate_field(np.asarray(f, float), t)


class CudaImpl:
    """B200 path through the C ABI (device-resident batch calls + host calls)."""

    def __init__(self, mode):
        import torch

        import paratime_b200 as B

        self.B = B
        self.torch = torch
        self.mode = mode
        self.name = "cuda-" + ("exact" if mode == B.EXACT else "fast")
        self.ctx = B.Context(0)

    def grid(self, n, h):
        return OracleImpl().grid(n, h)

    def _g(self, grid):
        return self.B.Grid(tuple(grid.n), tuple(grid.h))

    def laplacian(self, f, grid):
        f = np.asarray(f, dtype=np.float64)
        out = self.ctx.laplacian(self._g(grid), self.ctx.tensor(f))
        return out.cpu().numpy().reshape(f.shape)

    def _prop(self, grid, c, dt, steps):
        try:
            return self.B.Propagator(self.ctx, self._g(grid), np.asarray(c, float), dt, steps)
        except self.B.PtbError as e:
            if e.status == self.B.api.INVALID_ARGUMENT:
                raise InvalidArgument(str(e))
            raise

    def check_config(self, grid, c, dt, steps):
        self._prop(grid, c, dt, steps)

    def propagate(self, u, udot, c, grid, dt, steps):
        p = self._prop(grid, c, dt, steps)
        try:
            uo, vo = p.propagate_host(np.asarray(u, float).reshape(grid.shape),
                                      np.asarray(udot, float).reshape(grid.shape), mode=self.mode)
        except self.B.PtbError as e:
            if e.status == self.B.DIVERGED:
                raise Diverged(str(e))
            raise
        return uo, vo

    def propagate_batch(self, u, udot, c, grid, dt, steps, flags=False):
        p = self._prop(grid, c, dt, steps)
        tu, tv = self.ctx.tensor(u), self.ctx.tensor(udot)
        f = self.torch.zeros(tu.numel() // grid.size, dtype=self.torch.int32, device=tu.device) if flags else None
        p.propagate(tu, tv, mode=self.mode, flags=f)
        out = (tu.cpu().numpy(), tv.cpu().numpy())
        return out + (f.cpu().numpy(),) if flags else out

    def transfer(self, coarse, fine, kind):
        try:
            return self.B.Transfer(self.ctx, self._g(coarse), self._g(fine), kind)
        except self.B.PtbError as e:
            if e.status == self.B.api.INVALID_ARGUMENT:
                raise InvalidArgument(str(e))
            raise

    def restrict(self, f, t):
        f = np.asarray(f, float)
        out = t.restrict(self.ctx.tensor(f)).cpu().numpy()
        return out.reshape(f.shape[: f.ndim - t.fine.dim] + t.coarse.shape)

    def interpolate(self, f, t):
        f = np.asarray(f, float)
        out = t.interpolate(self.ctx.tensor(f)).cpu().numpy()
        return out.reshape(f.shape[: f.ndim - t.coarse.dim] + t.fine.shape)


# ---------------------------------------------------------------- energy / Procrustes / drivers

class Corr:
    """Uniform view of a corrector: X, S, Y (numpy) + the native handle."""

    def __init__(self, X, S, Y, native):
        self.X, self.S, self.Y, self.native = X, S, Y, native

    @property
    def rank(self):
        return self.S.shape[0]

    @property
    def rows(self):
        return self.X.shape[0]


def _oracle_corr(c):
    return Corr(c.X, c.S, c.Y, c)


class _OracleEnergy:
    def components(self, u, v, c, grid, scheme):
        s, m = P.to_energy_components(np.asarray(u, float), np.asarray(v, float), np.asarray(c, float), grid, scheme)
        return s, float(m) if np.ndim(m) == 0 else m

    def reconstruct(self, stacked, mean, c, grid):
        return P.from_energy_components(np.asarray(stacked, float), mean, np.asarray(c, float), grid)

    def energy(self, u, v, c, grid, scheme):
        return float(P.energy(np.asarray(u, float), np.asarray(v, float), np.asarray(c, float), grid, scheme))

    def energy_error(self, a, b, c, grid, scheme):
        return P.energy_error(a, b, np.asarray(c, float), grid, scheme)

    def procrustes_solve(self, F, G, tol):
        try:
            return _oracle_corr(P.procrustes_solve(F, G, tol))
        except ValueError as e:
            raise InvalidArgument(str(e))

    def update_svd(self, corr, F, G, tol):
        try:
            return _oracle_corr(P.update_svd(corr.native if corr is not None else P.empty_corrector(), F, G, tol))
        except ValueError as e:
            raise InvalidArgument(str(e))

    def relative_residual(self, corr, F, G):
        return P.relative_residual(corr.native, F, G)

    def drop_leading(self, corr, k):
        return _oracle_corr(corr.native.drop_leading(k))

    def apply(self, corr, v):
        return corr.native.apply(v)


for _name in dir(_OracleEnergy):
    if not _name.startswith("_"):
        setattr(OracleImpl, _name, getattr(_OracleEnergy, _name))


class _CudaEnergy:
    def _grid_dev(self, grid):
        return self._g(grid)

    def components(self, u, v, c, grid, scheme):
        u = np.asarray(u, float)
        B = self.B
        st, mean = B.api.energy_components(self.ctx, self._g(grid), self.ctx.tensor(c), scheme, self.ctx.tensor(u),
                                           self.ctx.tensor(v))
        st, mean = st.cpu().numpy(), mean.cpu().numpy()
        if u.shape == grid.shape:
            return st[0], float(mean[0])
        return st, mean

    def reconstruct(self, stacked, mean, c, grid):
        stacked = np.asarray(stacked, float)
        single = stacked.ndim == 1
        st = self.ctx.tensor(stacked.reshape(1, -1) if single else stacked)
        m = self.ctx.tensor(np.atleast_1d(np.asarray(mean, float)))
        u, v = self.B.api.from_energy_components(self.ctx, self._g(grid), self.ctx.tensor(c), st, m)
        u, v = u.cpu().numpy(), v.cpu().numpy()
        return (u[0], v[0]) if single else (u, v)

    def _sums(self, a, b, c, grid, scheme):
        t = self.ctx.tensor
        out = self.B.api.energy_sums(self.ctx, self._g(grid), t(c), scheme, t(a[0]), t(a[1]), t(b[0]), t(b[1]))
        return out.cpu().numpy()[0]

    def energy(self, u, v, c, grid, scheme):
        z = np.zeros_like(np.asarray(u, float))
        s = self._sums((np.asarray(u, float), np.asarray(v, float)), (z, z), c, grid, scheme)
        vol = float(np.prod(grid.h))
        return 0.5 * s[0] * vol

    def energy_error(self, a, b, c, grid, scheme):
        s = self._sums(a, b, c, grid, scheme)
        if s[1] == 0.0:
            raise ZeroDivisionError("energy_error: reference state has zero energy")
        return float(np.sqrt(s[0] / s[1]))

    def _corr(self, native):
        X, S, Y = native.factors()
        return Corr(X, S, Y, native)

    def _dev(self, M):
        return self.ctx.tensor(np.asarray(M, float).T.copy())  # (cols, rows) = column-major rows x cols

    def procrustes_solve(self, F, G, tol):
        c = self.B.api.Corrector(self.ctx)
        try:
            c.solve(self._dev(F), self._dev(G), tol)
        except self.B.PtbError as e:
            if e.status == self.B.api.INVALID_ARGUMENT:
                raise InvalidArgument(str(e))
            raise
        return self._corr(c)

    def update_svd(self, corr, F, G, tol):
        if corr is None:
            native = self.B.api.Corrector(self.ctx)
        else:  # update a copy (drop_leading(0)) so the input stays valid, like the value API
            native = corr.native.drop_leading(0)
        try:
            native.update(self._dev(F), self._dev(G), tol)
        except self.B.PtbError as e:
            if e.status == self.B.api.INVALID_ARGUMENT:
                raise InvalidArgument(str(e))
            raise
        return self._corr(native)

    def relative_residual(self, corr, F, G):
        return corr.native.residual(self._dev(F), self._dev(G))

    def drop_leading(self, corr, k):
        return self._corr(corr.native.drop_leading(k))

    def apply(self, corr, v):
        v = np.asarray(v, float)
        out = corr.native.apply(self.ctx.tensor(v.reshape(1, -1))).cpu().numpy()
        return out.reshape(v.shape)


for _name in dir(_CudaEnergy):
    if not _name.startswith("__"):
        setattr(CudaImpl, _name, getattr(_CudaEnergy, _name))
