"""Subprocess helper for tests/test_gpu_fullrow.py: FAST propagation on grids where k_wave2 can
run full-row strips (PTB_WAVE_FULL=2 forces them), against the oracle, plus the coupling ==
repeated single steps property (test_propagator.cpp:135-149)."""
import math
import sys

import numpy as np

import paratime_b200 as B
from oracle import paratime_np as P

ctx = B.Context(0)
worst = 0.0
plans = []
for (ny, nx), steps, batch in [((64, 192), 19, 3), ((40, 384), 8, 2), ((256, 256), 17, 2), ((24, 512), 9, 2)]:
    g = P.Grid((ny, nx), (1 / ny, 1 / nx))
    rng = np.random.default_rng(ny * nx)
    u = rng.uniform(-1, 1, (batch, ny, nx))
    v = rng.uniform(-1, 1, (batch, ny, nx))
    c = 0.5 + 0.5 * rng.random((ny, nx))
    dt = 0.9 * min(g.h) / (math.sqrt(2) * float(c.max()))
    ref = P.verlet_steps(u, v, c, g, dt, steps)
    prop = B.Propagator(ctx, B.Grid(g.n, g.h), c, dt, steps)
    plans.append(prop.plan(batch, B.FAST))
    tu, tv = ctx.tensor(u), ctx.tensor(v)
    prop.propagate(tu, tv, mode=B.FAST)
    got = np.concatenate([tu.cpu().numpy().ravel(), tv.cpu().numpy().ravel()])
    exp = np.concatenate([ref[0].ravel(), ref[1].ravel()])
    worst = max(worst, float(np.linalg.norm(got - exp) / np.linalg.norm(exp)))
    one = B.Propagator(ctx, B.Grid(g.n, g.h), c, dt, 1)
    su, sv = ctx.tensor(u), ctx.tensor(v)
    for _ in range(steps):
        one.propagate(su, sv, mode=B.FAST)
    if not (np.array_equal(su.cpu().numpy(), tu.cpu().numpy()) and np.array_equal(sv.cpu().numpy(), tv.cpu().numpy())):
        print("REPEAT_MISMATCH", ny, nx)
        sys.exit(1)
print("PLANS", " | ".join(plans))
print("WORST", worst)
