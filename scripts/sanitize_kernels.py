#!/usr/bin/env python
"""Workload for compute-sanitizer (racecheck / synccheck) over the kernels that use mbarriers,
st.async and DSMEM or grid barriers:
  k_wave2          - 512^2 / 256^2 slices (bulk-copy level-0 ring completing on mbarriers)
  k_cluster        - 128^2 slices (cluster of 8 CTAs, st.async halo rows + mbarrier tx counts)
  k_qr_panel       - truncated_qr of a 3072 x 96 block (blocked route: cooperative panel QR)
  k_jacobi_cluster - the 96 x 96 SVD of solve_from_scratch (8-CTA cluster, st.async all-gather)
plus the TSQR / register-QR / small Jacobi kernels that a config-1 sized update reaches.
  compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paratime_b200 as B  # noqa: E402

ctx = B.Context(0)
n = 128
rng = np.random.default_rng(1)
c = 0.75 + 0.25 * rng.random((n, n))
prop = B.Propagator(ctx, B.Grid((n, n), (1 / n, 1 / n)), c, 0.9 / n / (math.sqrt(2) * c.max()), 16)
print(prop.plan(2), flush=True)
u, v = ctx.tensor(rng.standard_normal((2, n, n))), ctx.tensor(np.zeros((2, n, n)))
prop.propagate(u, v, mode=B.FAST)
prop.propagate(u, v, mode=B.EXACT)
# k_wave2 (bulk-copy ring on mbarriers): a haloed-strip grid and a full-row grid
for n2 in (512, 256):
    c2 = 0.75 + 0.25 * rng.random((n2, n2))
    p2 = B.Propagator(ctx, B.Grid((n2, n2), (1 / n2, 1 / n2)), c2, 0.9 / n2 / (math.sqrt(2) * c2.max()), 8)
    print(p2.plan(2), flush=True)
    u2, v2 = ctx.tensor(rng.standard_normal((2, n2, n2))), ctx.tensor(np.zeros((2, n2, n2)))
    p2.propagate(u2, v2, mode=B.FAST)
for rows, cols in ((3072, 96), (3072, 16)):
    F = rng.standard_normal((cols, rows))  # device layout: (cols, rows) = column-major rows x cols
    G = F + 1e-2 * rng.standard_normal((cols, rows))
    co = B.api.Corrector(ctx)
    co.update(ctx.tensor(F), ctx.tensor(G), 1e-10)
    co.update(ctx.tensor(F[: cols // 2] * 1.1), ctx.tensor(G[: cols // 2]), 1e-10)
    print(rows, cols, co.shape(), flush=True)
ctx.synchronize()
print("sanitize workload done", flush=True)
