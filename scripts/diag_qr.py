#!/usr/bin/env python
"""Diagnostic: truncated_qr (procrustes.cpp:34-46) of the device on the first snapshot matrix F
of a real theta run (default config 3) vs LAPACK (oracle).  Stage 1 (no args beyond the path):
record F with the oracle; stage 2 (PTB_QR=<route> python diag_qr.py path run): factor it."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def record(path, cfg=3):
    import workloads as W
    from oracle import paratime_np as P
    from oracle import refbind
    from tests import configs as T

    spec, cf, cc, u0, v0 = W.CONFIGS[cfg]()

    def prop(u, udot, c, grid, dt, steps):
        uo, vo, _ = refbind.propagate(u, udot, c, grid, dt, steps, workers=16)
        return uo, vo

    P.propagate_coupling = prop
    P.fine_stage = lambda s, sch: prop(s[0], s[1], sch.c_fine, sch.fine_grid, sch.dt_fine, sch.m_fine)
    seen = []

    def rec(corr, F, G, tol):
        seen.append((F.copy(), G.copy()))
        raise StopIteration

    P.update_svd = rec
    fg = T.fine_grid(spec)
    cg = P.Grid(tuple(spec["coarse_n"]), tuple(spec["coarse_h"]))
    sch = P.Schedule(spec["T"], spec["dt_com"], spec["n_couplings"], fg, cf, spec["dt_fine"], spec["m_fine"], cg,
                     cc, spec["dt_coarse"], spec["m_coarse"])
    try:
        P.theta_parareal((u0, v0), sch, P.Transfer(cg, fg, spec["interp"]), 1, scheme=spec["scheme"], tol=spec["tol"])
    except StopIteration:
        pass
    np.savez(path, F=seen[0][0], G=seen[0][1])


def run(path):
    import torch

    import paratime_b200 as B
    from oracle import paratime_np as P

    d = np.load(path)
    ctx = B.Context(0)
    for name in ("F", "G"):
        a = d[name]
        m, n = a.shape
        A = torch.tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
        Q = torch.zeros(m * n, dtype=torch.float64, device="cuda")
        R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
        keep = C.c_size_t()
        tol = 1e-14 * np.linalg.norm(a)
        B.api.check(B.lib().ptb_truncated_qr(ctx.h, C.c_size_t(m), C.c_size_t(n), C.c_void_p(A.data_ptr()),
                                             C.c_double(tol), C.c_void_p(Q.data_ptr()), C.c_void_p(R.data_ptr()),
                                             C.byref(keep)))
        k = keep.value
        q = Q.cpu().numpy()[: m * k].reshape(k, m).T
        r = R.cpu().numpy()[: k * n].reshape(n, k).T
        qo, ro = P.truncated_qr(a, tol)
        sv = np.linalg.svd(a, compute_uv=False)
        print(f"{name}: keep dev {k} oracle {qo.shape[1]}  |QR-A|/|A| {np.linalg.norm(q @ r - a) / np.linalg.norm(a):.3e}"
              f"  orth {np.max(np.abs(q.T @ q - np.eye(k))):.3e}  |R^T R - Ro^T Ro|/|A|^2 "
              f"{np.linalg.norm(r.T @ r - ro.T @ ro) / np.linalg.norm(a) ** 2:.3e}  sv(A) min/max {sv[-1] / sv[0]:.3e}"
              f"  zero rows {int(np.sum(np.all(a == 0, axis=1)))}  min |a|>0 {np.min(np.abs(a[a != 0])):.3e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "run":
        run(sys.argv[1])
    else:
        record(sys.argv[1])
