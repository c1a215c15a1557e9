#!/usr/bin/env python
"""Scaled-down config 4 with its absorbing layer: plain vs theta parareal in the CPU oracle
(oracle/pml_np.py) — does the data-driven coupling stabilise the layered problem?
  python scripts/pml_theta_explore.py [nf] [nc] [width_f] [N] [K] [tol]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import workloads as W  # noqa: E402
from oracle import paratime_np as P  # noqa: E402
from oracle import pml_np as M  # noqa: E402

nf, nc, wf, N, K = (int(a) for a in (sys.argv[1:6] if len(sys.argv) > 5 else (256, 64, 16, 32, 6)))
tol = float(sys.argv[6]) if len(sys.argv) > 6 else 1e-4
r = nf // nc
rng = np.random.default_rng(W.SEED + 4)
c = W.layered_faulted(nf, rng)
cc = W.restrict(W.gaussian_smooth_periodic(c, r / 2), r)
y, x = W._mesh(nf)
x0 = rng.uniform(0.3, 0.7)
u0 = np.exp(-2500.0 * ((x - x0) ** 2 + (y - 0.15) ** 2))
v0 = np.zeros_like(u0)
cmax = float(c.max())
zf = M.damping_profile(nf, wf, 1 / nf, cmax)
zc = M.damping_profile(nc, wf // r, 1 / nc, cmax)
dtf, dtc = (1 / nf) / 8, (1 / nc) / 4
dtcom = 1.0 / N
mf, mc = round(dtcom / dtf), round(dtcom / dtc)
kf = M.PmlCoefficients(c, 1 / nf, 1 / nf, dtf, zf, zf)
kc = M.PmlCoefficients(cc, 1 / nc, 1 / nc, dtc, zc, zc)
t = P.Transfer(P.grid2(nc, nc, 1 / nc, 1 / nc), P.grid2(nf, nf, 1 / nf, 1 / nf), 0)
print(f"fine {nf}^2 layer {wf}, coarse {nc}^2, N={N} K={K} m_f={mf} m_c={mc} tol={tol}", flush=True)
variants = sys.argv[7].split(",") if len(sys.argv) > 7 else ["plain", "theta:plain", "theta:none"]
for var in variants:
    if var == "plain":
        _, e = M.plain_parareal(u0, v0, kf, mf, kc, mc, t, N, K)
        ranks = None
    else:
        _, e, ranks = M.theta_parareal(u0, v0, kf, mf, kc, mc, t, N, K, cc, tol=tol, aux=var.split(":")[1])
    print(f"{var:12s} max err per k:", " ".join(f"{x:.2e}" for x in e.max(axis=1)), "ranks", ranks, flush=True)
