#!/usr/bin/env python
"""Diagnostic: the device update_svd against the oracle's on the snapshot matrices of a real
theta run (default BASELINE config 3, first K iterations).  The oracle run records every (F, G)
its update_svd receives; the device corrector is fed the same sequence; factors and the action
of Omega = X Y^T are compared per iteration.
  python scripts/diag_procrustes.py [cfg=3] [K=3]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import workloads as W  # noqa: E402
from oracle import paratime_np as P  # noqa: E402
from oracle import refbind  # noqa: E402
from tests import configs as T  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec, cf, cc, u0, v0 = W.CONFIGS[cfg]()
spec["iterations"] = K


def prop(u, udot, c, grid, dt, steps):
    uo, vo, div = refbind.propagate(u, udot, c, grid, dt, steps, workers=16)
    return uo, vo


P.propagate_coupling = prop
P.fine_stage = lambda s, sch: prop(s[0], s[1], sch.c_fine, sch.fine_grid, sch.dt_fine, sch.m_fine)
seen = []
orig = P.update_svd


def rec(corr, F, G, tol):
    out = orig(corr, F, G, tol)
    seen.append((F.copy(), G.copy(), tol, out))
    return out


P.update_svd = rec
fg = T.fine_grid(spec)
cg = P.Grid(tuple(spec["coarse_n"]), tuple(spec["coarse_h"]))
sch = P.Schedule(spec["T"], spec["dt_com"], spec["n_couplings"], fg, cf, spec["dt_fine"], spec["m_fine"], cg, cc,
                 spec["dt_coarse"], spec["m_coarse"])
P.theta_parareal((u0, v0), sch, P.Transfer(cg, fg, spec["interp"]), K, scheme=spec["scheme"], tol=spec["tol"])

import paratime_b200 as B  # noqa: E402

ctx = B.Context(0)
corr = B.api.Corrector(ctx)
rng = np.random.default_rng(0)
for k, (F, G, tol, want) in enumerate(seen, 1):
    corr.update(ctx.tensor(np.ascontiguousarray(F.T)), ctx.tensor(np.ascontiguousarray(G.T)), tol)
    X, S, Y = corr.factors()
    v = rng.standard_normal(F.shape[0])
    om_g = X @ (Y.T @ v)
    om_o = want.X @ (want.Y.T @ v)
    print(f"k={k} F {F.shape} rank dev {X.shape[1]} oracle {want.X.shape[1]}  S rel {np.max(np.abs(S - want.S)) / want.S[0]:.3e}"
          f"  Omega v rel {np.linalg.norm(om_g - om_o) / np.linalg.norm(om_o):.3e}"
          f"  X col max {np.max(np.abs(np.abs(X) - np.abs(want.X))):.3e}  S[-3:] {want.S[-3:] / want.S[0]}", flush=True)
