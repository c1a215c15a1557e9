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
