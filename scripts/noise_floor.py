#!/usr/bin/env python
"""the oracle's own self-sensitivity floor per (config, tol, k).

The theta-parareal iterates amplify last-bit differences of the fine stage (continuous
sensitivity of the Procrustes singular vectors).  This script runs the oracle's
theta_parareal (oracle/paratime_np.py, parareal.cpp:255-350) twice per (config, tol): once
as is, once with every fine-stage output multiplied by (1 + eps*N(0,1)), eps = 1e-16 — the
size of the difference between the device's FMA-contracted FAST propagator and the
reference's (4.8e-15 relative after 64 steps).  The fine stage of both runs is
the reference's own propagate_coupling (oracle/_ref, propagator.cpp verbatim), so the
unperturbed run is the reference's arithmetic.  Output: max over n of energy_error(perturbed,
unperturbed) per k, the retained ranks of both runs, written to profiles/r02_noise_floor.json.

A GPU-vs-reference iterate distance below the floor is the best any implementation that is not
bitwise equal to the reference can claim; tests/test_gpu_configs.py asserts 1e-10 only where
the floor is <= 1e-11.

  python scripts/noise_floor.py [cfg ...]      (cfg in 1 2 3 4r; default all)
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import workloads as W  # noqa: E402
from oracle import paratime_np as P  # noqa: E402
from oracle import refbind  # noqa: E402
from tests import configs as T  # noqa: E402

EPS = 1e-16
CASES = {
    "1": (W.cfg1, (1e-8, 1e-13, 1e-15)),
    "2": (W.cfg2, (1e-4, 1e-6, 1e-10, 1e-13)),
    "3": (W.cfg3, (1e-4, 1e-6, 1e-10)),
    "4r": (T.reduced_cfg4, (1e-4,)),
}


def _install_fine_stage(rng):
    """P.fine_stage / P.propagate_coupling through the reference's own propagator, optionally
    perturbed (rng is None: exact reference arithmetic)."""

    def prop(u, udot, c, grid, dt, steps):
        uo, vo, div = refbind.propagate(u, udot, c, grid, dt, steps, workers=1)
        if div[0]:
            raise P.PropagationDiverged("non-finite")
        return uo[0] if uo.ndim > len(grid.shape) else uo, vo[0] if vo.ndim > len(grid.shape) else vo

    def fine(s, sch):
        try:
            u, v = prop(s[0], s[1], sch.c_fine, sch.fine_grid, sch.dt_fine, sch.m_fine)
        except P.PropagationDiverged:
            return P._nan_state(sch.fine_grid)
        if rng is not None:
            u = u * (1.0 + EPS * rng.standard_normal(u.shape))
            v = v * (1.0 + EPS * rng.standard_normal(v.shape))
        return u, v

    P.fine_stage = fine
    P.propagate_coupling = prop  # serial_fine reference and coarse stages: unperturbed


def run(cfg, tol, rng):
    spec, cf, cc, u0, v0 = CASES[cfg][0](tol=tol)
    _install_fine_stage(rng)
    fg = T.fine_grid(spec)
    cg = P.Grid(tuple(spec["coarse_n"]), tuple(spec["coarse_h"]))
    sch = P.Schedule(spec["T"], spec["dt_com"], spec["n_couplings"], fg, cf, spec["dt_fine"], spec["m_fine"], cg, cc,
                     spec["dt_coarse"], spec["m_coarse"])
    t = P.Transfer(cg, fg, spec["interp"])
    return P.theta_parareal((u0, v0), sch, t, spec["iterations"], scheme=spec["scheme"], tol=tol,
                            metric_scheme=spec["metric_scheme"]), cf, fg


def floor(cfg, tol):
    a, cf, fg = run(cfg, tol, None)
    b, _, _ = run(cfg, tol, np.random.default_rng(20261020))
    per_k = []
    for ra, rb in zip(a.iterations, b.iterations):
        worst = 0.0
        for n in range(1, len(ra.states)):
            x, y = ra.states[n], rb.states[n]
            if not (np.all(np.isfinite(x[0])) and np.all(np.isfinite(y[0]))):
                continue
            worst = max(worst, refbind.energy_error(y, x, cf, fg, 0))
        per_k.append(worst)
    return {"config": cfg, "tol": tol, "eps": EPS, "floor_per_k": per_k,
            "rank_unperturbed": [r.rank for r in a.iterations], "rank_perturbed": [r.rank for r in b.iterations]}


def main():
    cfgs = sys.argv[1:] or list(CASES)
    out_path = ROOT / "profiles" / "r02_noise_floor.json"
    results = json.loads(out_path.read_text()) if out_path.exists() else {}
    for cfg in cfgs:
        for tol in CASES[cfg][1]:
            t0 = time.time()
            r = floor(cfg, tol)
            r["seconds"] = round(time.time() - t0, 1)
            results[f"cfg{cfg} tol={tol:g}"] = r
            print(json.dumps(r), flush=True)
            out_path.write_text(json.dumps(results, indent=1) + "\n")


if __name__ == "__main__":
    main()
