"""Energy map, DFT, Procrustes and parareal drivers on the B200 vs the oracle.

Tolerances: finite-difference components/energies bitwise (reference operation order);
spectral/FFT maps 1e-12 relative (FFTW and the device FFT differ in round-off only);
corrector factors 1e-10; parareal iterates 1e-10 relative energy norm (north_star).
"""
import math

import numpy as np
import pytest

from oracle import paratime_np as P
from tests import kat

pytestmark = pytest.mark.gpu

ITERATE_TOL = 1e-10  # relative energy norm of iterates, north_star


@pytest.fixture(scope="module")
def impl():
    import paratime_b200 as B
    from tests.impls import CudaImpl

    return CudaImpl(B.FAST)


@pytest.mark.parametrize("check", kat.ENERGY_KATS + kat.PROCRUSTES_KATS, ids=lambda f: f.__name__)
def test_reference_known_answers_on_gpu(impl, check):
    check(impl)


GRIDS = [((36,), (1 / 36,)), ((12, 20), (1 / 12, 1 / 20)), ((32, 32), (1 / 32, 1 / 32)), ((48, 64), (0.02, 0.015)),
         ((9, 14), (0.1, 0.07))]


@pytest.mark.parametrize("gspec", GRIDS, ids=lambda g: "x".join(map(str, g[0])))
@pytest.mark.parametrize("scheme", [0, 1, 2, 3, 4])
def test_energy_components_parity(impl, gspec, scheme):
    g = P.Grid(*gspec)
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, (3,) + g.shape)
    v = rng.uniform(-1, 1, (3,) + g.shape)
    c = 0.5 + rng.random(g.shape)
    st_o, m_o = P.to_energy_components(u, v, c, g, scheme)
    st_g, m_g = impl.components(u, v, c, g, scheme)
    if scheme < 4:
        assert np.array_equal(st_g, st_o)
    else:
        assert np.max(np.abs(st_g - st_o)) <= 1e-12 * np.max(np.abs(st_o))
    assert np.max(np.abs(m_g - m_o)) <= 1e-13 * max(1.0, np.max(np.abs(m_o)))
    bu_o, bv_o = P.from_energy_components(st_o, m_o, c, g)
    bu_g, bv_g = impl.reconstruct(st_o, m_o, c, g)
    assert np.max(np.abs(bu_g - bu_o)) <= 1e-12 * np.max(np.abs(bu_o))
    assert np.array_equal(bv_g, bv_o)


@pytest.mark.parametrize("gspec", GRIDS, ids=lambda g: "x".join(map(str, g[0])))
@pytest.mark.parametrize("scheme", [0, 1, 4])
def test_energy_sums_parity(impl, gspec, scheme):
    g = P.Grid(*gspec)
    rng = np.random.default_rng(7)
    a = (rng.uniform(-1, 1, g.shape), rng.uniform(-1, 1, g.shape))
    b = (rng.uniform(-1, 1, g.shape), rng.uniform(-1, 1, g.shape))
    c = 0.5 + rng.random(g.shape)
    assert impl.energy_error(a, b, c, g, scheme) == pytest.approx(P.energy_error(a, b, c, g, scheme), rel=1e-13)
    assert impl.energy(a[0], a[1], c, g, scheme) == pytest.approx(float(P.energy(a[0], a[1], c, g, scheme)), rel=1e-13)


@pytest.mark.parametrize("shape", [(16,), (12,), (100,), (8, 16), (12, 20), (128, 128), (64, 256), (256, 64)])
def test_dft_matches_numpy(impl, shape, inverse=False):
    import paratime_b200 as B
    import torch

    rng = np.random.default_rng(1)
    z = rng.standard_normal((2,) + shape) + 1j * rng.standard_normal((2,) + shape)
    g = B.Grid(shape, tuple(1.0 / s for s in shape))
    for inv in (False, True):
        t = torch.as_tensor(z, device="cuda")
        B.api.dft(impl.ctx, g, t, inverse=inv)
        got = t.cpu().numpy()
        axes = tuple(range(1, 1 + len(shape)))
        ref = np.fft.ifftn(z, axes=axes) if inv else np.fft.fftn(z, axes=axes)
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref)) * math.log2(max(shape) + 1)


def test_procrustes_update_sequence_parity(impl):
    """A chained update_svd on snapshot-shaped data: device factors vs the oracle."""
    rng = np.random.default_rng(11)
    rows = 3 * 256
    co = P.empty_corrector()
    cg = None
    for k in range(4):
        F = rng.standard_normal((rows, 16))
        G = F + 1e-2 * rng.standard_normal((rows, 16))
        co = P.update_svd(co, F, G, 1e-10)
        cg = impl.update_svd(cg, F, G, 1e-10)
        assert cg.rank == co.rank
        assert np.max(np.abs(cg.S - co.S)) <= 1e-12 * co.S[0]
        assert np.max(np.abs(cg.X - co.X)) <= 1e-9
        assert np.max(np.abs(cg.Y - co.Y)) <= 1e-9
        assert impl.relative_residual(cg, F, G) == pytest.approx(P.relative_residual(co, F, G), rel=1e-10)


# ---------------------------------------------------------------- drivers


def config1(tol=1e-8, iterations=4, variant=1, scheme=0, interp=0, mode=0):
    """BASELINE config 1: 128^2 / 32^2, c = 1, N = 16, radial pulse exp(-400 r^2)."""
    n, nc = 128, 32
    y, x = np.meshgrid(np.arange(n) / n, np.arange(n) / n, indexing="ij")
    u0 = np.exp(-400.0 * ((x - 0.5) ** 2 + (y - 0.5) ** 2))
    spec = dict(dim=2, fine_n=(n, n), fine_h=(1 / n, 1 / n), coarse_n=(nc, nc), coarse_h=(1 / nc, 1 / nc),
                dt_fine=0.0625 / 64, m_fine=64, dt_coarse=0.0625 / 8, m_coarse=8, T=1.0, dt_com=0.0625,
                n_couplings=16, interp=interp, iterations=iterations, variant=variant, scheme=scheme,
                metric_scheme=scheme, tol=tol, remove_leading=0, mode=mode)
    return spec, np.ones((n, n)), np.ones((nc, nc)), u0, np.zeros_like(u0)


def run_gpu(spec, cf, cc, u0, v0, **kw):
    import paratime_b200 as B

    ctx = B.Context(0)
    return B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, **kw)


def run_oracle(spec, cf, cc, u0, v0):
    fg = P.Grid(tuple(spec["fine_n"][: spec["dim"]]), tuple(spec["fine_h"][: spec["dim"]]))
    cgr = P.Grid(tuple(spec["coarse_n"][: spec["dim"]]), tuple(spec["coarse_h"][: spec["dim"]]))
    sch = P.Schedule(spec["T"], spec["dt_com"], spec["n_couplings"], fg, cf.reshape(fg.shape), spec["dt_fine"],
                     spec["m_fine"], cgr, cc.reshape(cgr.shape), spec["dt_coarse"], spec["m_coarse"])
    t = P.Transfer(cgr, fg, spec["interp"])
    init = (u0.reshape(fg.shape), v0.reshape(fg.shape))
    if spec["variant"] == 0:
        run = P.plain_parareal(init, sch, t, spec["iterations"], metric_scheme=spec["metric_scheme"])
    else:
        run = P.theta_parareal(init, sch, t, spec["iterations"], scheme=spec["scheme"], tol=spec["tol"],
                               omega_identity=spec["variant"] == 3, additive_correction=spec["variant"] != 2,
                               remove_leading=spec["remove_leading"], metric_scheme=spec["metric_scheme"])
    return run, fg


def compare(gpu, run, fg, cf, scheme=0, tol=ITERATE_TOL):
    worst = 0.0
    for k, rec in enumerate(run.iterations):
        for n, (u, v) in enumerate(rec.states):
            gu, gv = gpu["states"][k, n]
            if not (np.all(np.isfinite(u)) and np.all(np.isfinite(v))):
                assert not np.all(np.isfinite(gu))
                continue
            if float(P.energy(u, v, cf.reshape(fg.shape), fg, scheme)) == 0.0:
                assert np.max(np.abs(gu - u)) <= 1e-14
                continue
            worst = max(worst, P.energy_error((gu, gv), (u, v), cf.reshape(fg.shape), fg, scheme))
        assert list(gpu["rank"][1:]) == [r.rank for r in run.iterations[1:]]
        np.testing.assert_allclose(gpu["energy_err"][k], rec.energy_err, rtol=1e-6, atol=1e-12)
    assert worst <= tol, worst
    return worst


@pytest.mark.parametrize("mode", [0, 1])
def test_theta_config1_matches_oracle(mode):
    spec, cf, cc, u0, v0 = config1(tol=1e-8, mode=mode)
    gpu = run_gpu(spec, cf, cc, u0, v0, keep_states=True)
    run, fg = run_oracle(spec, cf, cc, u0, v0)
    compare(gpu, run, fg, cf)
    assert np.all(np.isfinite(gpu["residual"][1:]))


def test_plain_config1_matches_oracle():
    spec, cf, cc, u0, v0 = config1(variant=0)
    gpu = run_gpu(spec, cf, cc, u0, v0, keep_states=True)
    run, fg = run_oracle(spec, cf, cc, u0, v0)
    compare(gpu, run, fg, cf)


@pytest.mark.parametrize("variant,interp,scheme", [(1, 1, 1), (2, 0, 1), (3, 0, 4), (1, 0, 4)])
def test_variants_config1_match_oracle(variant, interp, scheme):
    spec, cf, cc, u0, v0 = config1(tol=1e-6, iterations=3, variant=variant, interp=interp, scheme=scheme)
    gpu = run_gpu(spec, cf, cc, u0, v0, keep_states=True)
    run, fg = run_oracle(spec, cf, cc, u0, v0)
    compare(gpu, run, fg, cf, scheme=scheme)


def test_theta_exact_at_couplings_n_le_k():
    """test_parareal.cpp:116-131 / acceptance criterion 1 on config 1."""
    spec, cf, cc, u0, v0 = config1(tol=1e-8, iterations=4)
    gpu = run_gpu(spec, cf, cc, u0, v0)
    for k in range(5):
        assert np.all(gpu["energy_err"][k, : k + 1] <= 1e-10)


def test_nonfinite_initial_state_flags_divergence():
    """test_parareal.cpp:182-194."""
    spec, cf, cc, u0, v0 = config1(iterations=2)
    u0 = u0.copy()
    u0[0, 0] = np.nan
    gpu = run_gpu(spec, cf, cc, u0, v0)
    assert gpu["diverged"][0] == 1
    assert np.all(np.isinf(gpu["energy_err"][:, -1]))


@pytest.mark.parametrize("variant", [0, 1])
def test_overflowing_iterates_flag_divergence(variant):
    """A finite initial state whose propagation overflows (amplitude 1e305): every state after
    the first is non-finite, so the per-iteration divergence flags come from the finalize error
    sums of states 1..N (parareal.cpp:107-128), not from the state-0 check.  EXACT mode: it
    follows the reference's operation order, so it overflows where the reference does (FAST
    mode's premultiplied kick coefficient keeps these states finite)."""
    spec, cf, cc, u0, v0 = config1(iterations=2, variant=variant, mode=1)
    u0 = u0 * 1e305
    gpu = run_gpu(spec, cf, cc, u0, v0)
    with np.errstate(over="ignore", invalid="ignore"):
        run, _ = run_oracle(spec, cf, cc, u0, v0)
    assert list(gpu["diverged"]) == [int(r.diverged) for r in run.iterations] == [1, 1, 1]
    for k, rec in enumerate(run.iterations):
        np.testing.assert_array_equal(gpu["energy_err"][k], rec.energy_err)


def test_overflowing_iterates_flag_divergence_wide_grid():
    """Same on config 2's 256^2 fine grid (the 2-D error-sum kernel)."""
    import workloads as W

    spec, cf, cc, u0, v0 = W.cfg2(mode=1)
    spec["iterations"] = 2
    gpu = run_gpu(spec, cf, cc, u0 * 1e305, v0)
    assert list(gpu["diverged"]) == [1, 1, 1]
    assert np.all(gpu["energy_err"][:, 0] == 0.0)
    assert np.all(np.isinf(gpu["energy_err"][:, 1:]))


def test_one_dimensional_preset_matches_reference(ref):
    """The reference's own rank-tolerance preset (experiment.cpp:279-284), shortened."""
    spec_r, cf, cc, u0, v0 = ref.build_setup("rank-tolerance", overrides="iterations=4\nT=2")
    r = ref.parareal_run(spec_r, cf, cc, u0, v0, keep_states=True)
    spec = dict(dim=1, fine_n=(spec_r.fine_n[0],), fine_h=(spec_r.fine_h[0],), coarse_n=(spec_r.coarse_n[0],),
                coarse_h=(spec_r.coarse_h[0],), dt_fine=spec_r.dt_fine, m_fine=spec_r.m_fine,
                dt_coarse=spec_r.dt_coarse, m_coarse=spec_r.m_coarse, T=spec_r.T, dt_com=spec_r.dt_com,
                n_couplings=spec_r.n_couplings, interp=spec_r.interp, iterations=spec_r.iterations,
                variant=spec_r.variant, scheme=spec_r.scheme, metric_scheme=spec_r.metric_scheme, tol=1e-8,
                remove_leading=0, mode=1)
    spec_r.tol = 1e-8
    r = ref.parareal_run(spec_r, cf, cc, u0, v0, keep_states=True)
    gpu = run_gpu(spec, cf, cc, u0, v0, keep_states=True)
    fg = P.Grid((spec_r.fine_n[0],), (spec_r.fine_h[0],))
    worst = 0.0
    for k in range(spec["iterations"] + 1):
        for n in range(1, spec["n_couplings"] + 1):
            a = gpu["states"][k, n]
            b = r["states"][k, n]
            worst = max(worst, P.energy_error((a[0], a[1]), (b[0], b[1]), cf, fg, 0))
    assert list(gpu["rank"]) == list(r["rank"])
    assert worst <= ITERATE_TOL, worst


@pytest.mark.parametrize("shape", [(256, 256), (128, 512), (512, 256)])
@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_streaming_pair_sums_match_row_kernel(impl, shape, scheme, monkeypatch):
    """k_pair_sums_stream (column windows in registers, the default on nx % 256 == 0) against the
    row-per-block k_pair_sums2d and the oracle: the same per-point arithmetic, only the grouping
    of the partial sums differs."""
    g = P.Grid(shape, (1.0 / shape[0], 1.0 / shape[1]))
    rng = np.random.default_rng(11)
    a = (rng.uniform(-1, 1, g.shape), rng.uniform(-1, 1, g.shape))
    b = (rng.uniform(-1, 1, g.shape), rng.uniform(-1, 1, g.shape))
    c = 0.5 + rng.random(g.shape)
    got = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("PTB_PAIR_STREAM", mode)
        got[mode] = impl.energy_error(a, b, c, g, scheme)
    want = P.energy_error(a, b, c, g, scheme)
    assert got["1"] == pytest.approx(want, rel=1e-13)
    assert got["1"] == pytest.approx(got["0"], rel=1e-13)
