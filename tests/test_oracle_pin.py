"""Pin the numpy oracle to the reference: against the golden fixtures generated from the
reference itself (tests/golden, always available) and, when oracle/_ref can be built or is
shipped, against the live reference library on fresh random inputs."""
from pathlib import Path

import numpy as np
import pytest

from oracle import paratime_np as P

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "reference_fixtures.npz")


def test_propagator_bitwise_vs_reference_fixtures():
    g2 = P.Grid((24, 20), (1 / 24, 1 / 20))
    u, v = P.verlet_steps(GOLD["p2_u0"], GOLD["p2_v0"], GOLD["p2_c"], g2, float(GOLD["p2_dt"]), int(GOLD["p2_steps"]))
    assert np.array_equal(u, GOLD["p2_u"]) and np.array_equal(v, GOLD["p2_v"])
    g1 = P.Grid((50,), (0.02,))
    u, v = P.verlet_steps(GOLD["p1_u0"], GOLD["p1_v0"], np.ones(50), g1, 0.01, 9)
    assert np.array_equal(u, GOLD["p1_u"]) and np.array_equal(v, GOLD["p1_v"])


def test_transfer_vs_reference_fixtures():
    cg, fg = P.Grid((6, 10), (0.25, 0.1)), P.Grid((18, 30), (0.25 / 3, 0.1 / 3))
    f = GOLD["t_coarse"]
    assert np.array_equal(P.interpolate_field(f, P.Transfer(cg, fg, P.LINEAR)), GOLD["t_linear"])
    assert np.max(np.abs(P.interpolate_field(f, P.Transfer(cg, fg, P.FOURIER)) - GOLD["t_fourier"])) <= 1e-14


@pytest.mark.parametrize("scheme", [0, 1, 4])
def test_energy_map_vs_reference_fixtures(scheme):
    g = P.Grid((12, 16), (1 / 12, 1 / 16))
    st, mean = P.to_energy_components(GOLD["e_u"], GOLD["e_v"], GOLD["e_c"], g, scheme)
    ref = GOLD[f"e_stack{scheme}"]
    if scheme < 4:
        assert np.array_equal(st, ref)
        assert float(P.energy(GOLD["e_u"], GOLD["e_v"], GOLD["e_c"], g, scheme)) == float(GOLD[f"e_energy{scheme}"])
    else:
        assert np.max(np.abs(st - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert abs(float(mean) - float(GOLD[f"e_mean{scheme}"])) <= 1e-13 * max(1.0, abs(float(GOLD[f"e_mean{scheme}"])))
    bu, bv = P.from_energy_components(ref, float(GOLD[f"e_mean{scheme}"]), GOLD["e_c"], g)
    assert np.max(np.abs(bu - GOLD[f"e_back{scheme}_u"])) <= 1e-13
    assert np.array_equal(bv, GOLD[f"e_back{scheme}_v"])


def test_procrustes_vs_reference_fixtures():
    c = P.empty_corrector()
    for k in range(3):
        c = P.update_svd(c, GOLD[f"q_F{k}"], GOLD[f"q_G{k}"], 1e-12)
        assert np.max(np.abs(c.S - GOLD[f"q_S{k}"])) <= 1e-12 * GOLD[f"q_S{k}"][0]
        assert np.max(np.abs(c.X - GOLD[f"q_X{k}"])) <= 1e-10
        assert np.max(np.abs(c.Y - GOLD[f"q_Y{k}"])) <= 1e-10
        assert P.relative_residual(c, GOLD[f"q_F{k}"], GOLD[f"q_G{k}"]) == pytest.approx(float(GOLD[f"q_res{k}"]), rel=1e-10)


def test_theta_config1_vs_reference_fixtures():
    import workloads as W

    spec, cf, cc, u0, v0 = W.cfg1(tol=1e-8)
    fg, cgr = P.Grid((128, 128), (1 / 128, 1 / 128)), P.Grid((32, 32), (1 / 32, 1 / 32))
    sch = P.Schedule(1.0, 0.0625, 16, fg, cf, spec["dt_fine"], 64, cgr, cc, spec["dt_coarse"], 8)
    run = P.theta_parareal((u0, v0), sch, P.Transfer(cgr, fg, P.FOURIER), 4, scheme=0, tol=1e-8)
    assert [r.rank for r in run.iterations] == list(GOLD["d1_rank"])
    ee = np.array([r.energy_err for r in run.iterations])
    np.testing.assert_allclose(ee, GOLD["d1_energy_err"], rtol=1e-8, atol=1e-12)
    fu, fv = run.iterations[-1].states[-1]
    assert P.energy_error((fu, fv), (GOLD["d1_final"][0], GOLD["d1_final"][1]), cf, fg, 0) <= 1e-10


def test_live_reference_propagator_and_drivers(ref):
    """Fresh inputs through the live reference library (oracle/_ref)."""
    rng = np.random.default_rng(99)
    g = P.Grid((40, 36), (1 / 40, 1 / 36))
    c = 0.6 + 0.4 * rng.random(g.shape)
    u, v = rng.uniform(-1, 1, (3,) + g.shape), rng.uniform(-1, 1, (3,) + g.shape)
    a = P.verlet_steps(u, v, c, g, 0.004, 21)
    b = ref.propagate(u, v, c, g, 0.004, 21, workers=3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for s in range(5):
        x = P.to_energy_components(u[0], v[0], c, g, s)[0]
        y = ref.energy_components(u[0], v[0], c, g, s)[0]
        assert (np.array_equal(x, y) if s < 4 else np.max(np.abs(x - y)) <= 1e-12 * np.max(np.abs(y)))
