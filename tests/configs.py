"""Shared helpers for the BASELINE-config parity tests (test infrastructure).

`reference_run` drives the reference's own theta_parareal / plain_parareal (oracle/_ref:
parareal.cpp compiled verbatim, Procrustes restated on LAPACK) on a workloads.py spec;
`iterate_distance` measures GPU-vs-reference iterates with the reference's metrics
(energy_error, energy_map.cpp:228-236; l2_error, :238-249).
"""
from __future__ import annotations

import os

import numpy as np

import workloads as W
from oracle import paratime_np as P

SPEC_KEYS = ("dt_fine", "m_fine", "dt_coarse", "m_coarse", "T", "dt_com", "n_couplings", "interp", "iterations",
             "variant", "scheme", "metric_scheme", "tol", "remove_leading")


reduced_cfg4 = W.cfg4_subset


def ref_spec(ref, spec, workers=None):
    rs = ref.RunSpec()
    rs.dim = spec["dim"]
    for k in range(spec["dim"]):
        rs.fine_n[k], rs.fine_h[k] = spec["fine_n"][k], spec["fine_h"][k]
        rs.coarse_n[k], rs.coarse_h[k] = spec["coarse_n"][k], spec["coarse_h"][k]
    for k in SPEC_KEYS:
        setattr(rs, k, spec[k])
    rs.workers = workers or (os.cpu_count() or 1)
    return rs


def reference_run(ref, spec, cf, cc, u0, v0, keep_states=True, workers=None):
    return ref.parareal_run(ref_spec(ref, spec, workers), cf, cc, u0, v0, keep_states=keep_states)


def fine_grid(spec):
    d = spec["dim"]
    return P.Grid(tuple(spec["fine_n"][:d]), tuple(spec["fine_h"][:d]))


def iterate_distance(ref, gpu_states, ref_states, cf, grid, scheme=0):
    """max over (k, n) of energy_error(gpu, ref) and l2_error(gpu.u, ref.u) — the north star's
    iterate criterion (relative energy norm) plus the l2 check the energy seminorm needs (it is
    blind to a constant offset in u), both evaluated by the reference's own code (oracle/_ref).
    States are (K+1, N+1, 2, *grid)."""
    K1, N1 = ref_states.shape[:2]
    ee = np.zeros((K1, N1))
    l2 = np.zeros((K1, N1))
    c = cf.reshape(grid.shape)
    for k in range(K1):
        for n in range(1, N1):
            a, b = gpu_states[k, n], ref_states[k, n]
            if not (np.all(np.isfinite(b)) and np.all(np.isfinite(a))):
                ee[k, n] = l2[k, n] = np.inf
                continue
            ee[k, n] = ref.energy_error((a[0], a[1]), (b[0], b[1]), c, grid, scheme)
            l2[k, n] = ref.l2_error(a[0], b[0], grid)
    return ee, l2
