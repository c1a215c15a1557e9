"""Fine-state parity of the exact kernel plans the benchmark times (north star: <= 1e-12
relative L2 over [u; udot] against the reference's propagate_coupling, propagator.cpp:95-105,
compiled verbatim in oracle/_ref).

Every (grid, batch) below is a line of bench.py (the headline 4096^2 x 512 and the cfg5 sweep)
or a fine stage of the parareal configs; the device runs the WHOLE batch, so the planner picks
the same strip width / full-row / ry1 / row-block / scratch-chunk variant as the timed run,
and a spread of slices (first, last, between) is compared with the reference on identical
inputs.  The plan string is asserted to be the one the bench line reports."""
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle.paratime_np import Grid

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-12

CASES = [  # (grid, batch, steps, expected plan fragment)
    (128, 64, 64, "k_cluster"),
    (128, 512, 64, "full-row ry1"),
    (256, 64, 64, "ry1"),
    (512, 64, 64, "ry1"),
    (1024, 64, 64, "ry1"),
    (2048, 64, 64, "ry1"),
    (2048, 128, 128, "ry1"),  # config 4's fine stage on one GPU (N = 128, m_F = 128)
    (4096, 64, 64, "ry1"),
    (4096, 512, 64, "per chunk of"),  # the headline: 137 GB of state, chunked ping-pong scratch
]


def _slices(batch, k):
    return sorted({int(round(i * (batch - 1) / (k - 1))) for i in range(k)})


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}^2x{c[1]}-m{c[2]}")
def test_bench_plan_matches_reference(ref, case):
    import torch

    import paratime_b200 as B

    n, batch, steps, frag = case
    ctx = B.Context(0)
    c = W.cfg5_medium(n)
    dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
    prop = B.Propagator(ctx, B.Grid((n, n), (1.0 / n, 1.0 / n)), c, dt, steps)
    plan = prop.plan(batch, B.FAST)
    assert frag in plan, plan
    u = torch.empty((batch, n, n), dtype=torch.float64, device="cuda")
    W.cfg5_pulses_device(n, batch, u)
    v = torch.zeros_like(u)
    idx = _slices(batch, 4 if n >= 2048 else 8)
    u0 = u[idx].cpu().numpy()
    flags = torch.zeros(batch, dtype=torch.int32, device="cuda")
    prop.propagate(u, v, mode=B.FAST, flags=flags)
    got_u, got_v = u[idx].cpu().numpy(), v[idx].cpu().numpy()
    assert int(flags.sum()) == 0
    del u, v
    torch.cuda.empty_cache()
    ru, rv, div = ref.propagate(u0, np.zeros_like(u0), c, Grid((n, n), (1.0 / n, 1.0 / n)), dt, steps,
                                workers=os.cpu_count() or 1)
    assert not div.any()
    for b in range(len(idx)):
        num = np.concatenate([got_u[b].ravel() - ru[b].ravel(), got_v[b].ravel() - rv[b].ravel()])
        den = np.concatenate([ru[b].ravel(), rv[b].ravel()])
        assert np.linalg.norm(num) / np.linalg.norm(den) <= FAST_TOL, (idx[b], plan)
