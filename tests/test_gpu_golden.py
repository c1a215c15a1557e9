"""The device path against fixtures generated from the reference itself (tests/golden)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import paratime_np as P

pytestmark = pytest.mark.gpu

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "reference_fixtures.npz")


@pytest.fixture(scope="module")
def B():
    import paratime_b200

    return paratime_b200


@pytest.fixture(scope="module")
def ctx(B):
    return B.Context(0)


def test_exact_propagator_bitwise_vs_reference(B, ctx):
    p = B.Propagator(ctx, B.Grid((24, 20), (1 / 24, 1 / 20)), GOLD["p2_c"], float(GOLD["p2_dt"]), int(GOLD["p2_steps"]))
    u, v = ctx.tensor(GOLD["p2_u0"]), ctx.tensor(GOLD["p2_v0"])
    p.propagate(u, v, mode=B.EXACT)
    assert np.array_equal(u.cpu().numpy(), GOLD["p2_u"]) and np.array_equal(v.cpu().numpy(), GOLD["p2_v"])
    p1 = B.Propagator(ctx, B.Grid((50,), (0.02,)), np.ones(50), 0.01, 9)
    uo, vo = p1.propagate_host(GOLD["p1_u0"], GOLD["p1_v0"], mode=B.EXACT)
    assert np.array_equal(uo, GOLD["p1_u"]) and np.array_equal(vo, GOLD["p1_v"])


def test_fast_propagator_within_1e12_vs_reference(B, ctx):
    p = B.Propagator(ctx, B.Grid((24, 20), (1 / 24, 1 / 20)), GOLD["p2_c"], float(GOLD["p2_dt"]), int(GOLD["p2_steps"]))
    u, v = ctx.tensor(GOLD["p2_u0"]), ctx.tensor(GOLD["p2_v0"])
    p.propagate(u, v, mode=B.FAST)
    for b in range(2):
        got = np.concatenate([u.cpu().numpy()[b].ravel(), v.cpu().numpy()[b].ravel()])
        ref = np.concatenate([GOLD["p2_u"][b].ravel(), GOLD["p2_v"][b].ravel()])
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12


def test_transfer_vs_reference(B, ctx):
    cg, fg = B.Grid((6, 10), (0.25, 0.1)), B.Grid((18, 30), (0.25 / 3, 0.1 / 3))
    f = ctx.tensor(GOLD["t_coarse"])
    assert np.array_equal(B.Transfer(ctx, cg, fg, B.LINEAR).interpolate(f).cpu().numpy()[0], GOLD["t_linear"])
    four = B.Transfer(ctx, cg, fg, B.FOURIER).interpolate(f).cpu().numpy()[0]
    assert np.max(np.abs(four - GOLD["t_fourier"])) <= 1e-14


@pytest.mark.parametrize("scheme", [0, 1, 4])
def test_energy_map_vs_reference(B, ctx, scheme):
    g = B.Grid((12, 16), (1 / 12, 1 / 16))
    c = ctx.tensor(GOLD["e_c"])
    st, mean = B.api.energy_components(ctx, g, c, scheme, ctx.tensor(GOLD["e_u"]), ctx.tensor(GOLD["e_v"]))
    ref = GOLD[f"e_stack{scheme}"]
    if scheme < 4:
        assert np.array_equal(st.cpu().numpy()[0], ref)
    else:
        assert np.max(np.abs(st.cpu().numpy()[0] - ref)) <= 1e-12 * np.max(np.abs(ref))
    u, v = B.api.from_energy_components(ctx, g, c, ctx.tensor(ref[None]), ctx.tensor([float(GOLD[f"e_mean{scheme}"])]))
    assert np.max(np.abs(u.cpu().numpy()[0] - GOLD[f"e_back{scheme}_u"])) <= 1e-13
    assert np.array_equal(v.cpu().numpy()[0], GOLD[f"e_back{scheme}_v"])


def test_procrustes_vs_reference(B, ctx):
    c = B.api.Corrector(ctx)
    for k in range(3):
        F, G = GOLD[f"q_F{k}"], GOLD[f"q_G{k}"]
        c.update(ctx.tensor(F.T.copy()), ctx.tensor(G.T.copy()), 1e-12)
        X, S, Y = c.factors()
        assert np.max(np.abs(S - GOLD[f"q_S{k}"])) <= 1e-12 * GOLD[f"q_S{k}"][0]
        assert np.max(np.abs(X - GOLD[f"q_X{k}"])) <= 1e-10
        assert np.max(np.abs(Y - GOLD[f"q_Y{k}"])) <= 1e-10
        assert c.residual(ctx.tensor(F.T.copy()), ctx.tensor(G.T.copy())) == pytest.approx(float(GOLD[f"q_res{k}"]),
                                                                                           rel=1e-10)


@pytest.mark.parametrize("mode", [0, 1])
def test_theta_config1_vs_reference(B, ctx, mode):
    import workloads as W

    spec, cf, cc, u0, v0 = W.cfg1(tol=1e-8, mode=mode)
    r = B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, keep_states=True)
    assert list(r["rank"]) == list(GOLD["d1_rank"])
    np.testing.assert_allclose(r["energy_err"], GOLD["d1_energy_err"], rtol=1e-8, atol=1e-12)
    fg = P.Grid((128, 128), (1 / 128, 1 / 128))
    for got, ref in ((r["states"][-1, -1], GOLD["d1_final"]), (r["states"][2, 8], GOLD["d1_mid"])):
        assert P.energy_error((got[0], got[1]), (ref[0], ref[1]), cf, fg, 0) <= 1e-10


def test_rank_tolerance_preset_vs_reference(B, ctx):
    s = GOLD["d2_spec"]
    spec = dict(dim=1, fine_n=(int(s[0]),), fine_h=(float(s[1]),), coarse_n=(int(s[2]),), coarse_h=(float(s[3]),),
                dt_fine=float(s[4]), m_fine=int(s[5]), dt_coarse=float(s[6]), m_coarse=int(s[7]), T=float(s[8]),
                dt_com=float(s[9]), n_couplings=int(s[10]), interp=int(s[11]), iterations=int(s[12]),
                variant=int(s[13]), scheme=int(s[14]), metric_scheme=int(s[14]), tol=1e-8, remove_leading=0, mode=1)
    r = B.api.parareal_run(ctx, B.api.run_spec(**spec), GOLD["d2_c"], GOLD["d2_c"], GOLD["d2_u0"],
                           np.zeros_like(GOLD["d2_u0"]), keep_states=True)
    assert list(r["rank"]) == list(GOLD["d2_rank"])
    fg = P.Grid((int(s[0]),), (float(s[1]),))
    fin = r["states"][-1, -1]
    assert P.energy_error((fin[0], fin[1]), (GOLD["d2_final"][0], GOLD["d2_final"][1]), GOLD["d2_c"], fg, 0) <= 1e-10
