"""Absorbing-layer (PML) oracle: self-consistency pins (CPU only).

The reference has no absorbing layer (propagator.cpp:31-105 is periodic),
so oracle/pml_np.py is pinned by properties instead of by reference outputs ("parity unpinned"):
zero profile == the periodic propagator, absorption against a boundary-free run on a 3x larger
periodic box, stability, and the host profile of the C ABI equal to the oracle's bitwise."""
import numpy as np
import pytest

from oracle import paratime_np as P
from oracle import pml_np as M


def _pulse(n, w=400.0, x0=0.5, y0=0.5, extent=1.0):
    y, x = np.meshgrid(np.arange(n) * (extent / n), np.arange(n) * (extent / n), indexing="ij")
    return np.exp(-w * ((x - x0) ** 2 + (y - y0) ** 2))


def test_zero_profile_is_the_periodic_propagator():
    n, h = 48, 1 / 48
    rng = np.random.default_rng(1)
    c = 0.6 + 0.4 * rng.random((n, n))
    u, v = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    k = M.PmlCoefficients(c, h, h, h / 8, np.zeros(n), np.zeros(n))
    z = np.zeros((n, n))
    a = M.pml_steps(u, v, z, z, k, 40)
    r = P.verlet_steps(u[None], v[None], c, P.Grid((n, n), (h, h)), h / 8, 40)
    for got, want in ((a[0], r[0][0]), (a[1], r[1][0])):
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    assert not a[2].any() and not a[3].any()  # auxiliary fields stay zero without a layer


def test_profile_shape():
    z = M.damping_profile(64, 8, 1 / 64, 1.0, 1e-4)
    assert np.all(z[8:56] == 0.0) and np.all(z[:8] > 0)
    assert np.array_equal(z[:8], z[::-1][:8])  # symmetric
    assert np.all(np.diff(z[:8]) < 0)  # deepest cell (the box edge) damps most
    with pytest.raises(ValueError):
        M.damping_profile(16, 8, 1 / 16, 1.0)


@pytest.mark.parametrize("aspect", [1.0, 0.5])
def test_pulse_is_absorbed(aspect):
    n, W = 96, 12
    hx = 1 / n
    hy = hx * aspect
    dt = hy / 8
    c = np.ones((n, n))
    u0 = _pulse(n, w=600.0)
    z = np.zeros((n, n))
    zy = M.damping_profile(n, W, hy, 1.0, 1e-3)
    zx = M.damping_profile(n, W, hx, 1.0, 1e-3)
    k = M.PmlCoefficients(c, hy, hx, dt, zy, zx)
    # boundary-free reference: the same pulse on a 3x larger periodic box (no reflection arrives
    # in the interior window before t = 1/c)
    N3 = 3 * n
    U = np.zeros((N3, N3))
    U[n:2 * n, n:2 * n] = u0
    g3 = P.Grid((N3, N3), (hy, hx))
    e0 = M.interior_energy(u0, z, c, hy, hx, W)
    s, S = (u0, z, z, z), (U[None], np.zeros((1, N3, N3)))
    errs, energies = [], []
    for _ in range(16):  # 16 x 48 steps (t = 1): the pulse crosses the layer
        s = M.pml_steps(*s, k, 48)
        S = P.verlet_steps(S[0], S[1], np.ones((N3, N3)), g3, dt, 48)
        ref = S[0][0][n:2 * n, n:2 * n]
        errs.append(float(np.max(np.abs(s[0] - ref)[W:n - W, W:n - W])))
        energies.append(M.interior_energy(s[0], s[1], c, hy, hx, W) / e0)
    assert max(errs) < 5e-3, errs  # reflected amplitude vs a pulse of amplitude 1
    assert all(np.isfinite(errs))
    if aspect == 1.0:
        assert energies[-1] < 0.05, energies  # the energy has left through the layer


def test_stable_over_long_runs():
    n, W = 64, 10
    h = 1 / n
    rng = np.random.default_rng(3)
    c = 0.5 + 0.5 * rng.random((n, n))
    zs = M.damping_profile(n, W, h, 1.0, 1e-6)
    k = M.PmlCoefficients(c, h, h, h / 8, zs, zs)
    u = rng.standard_normal((n, n))
    z = np.zeros((n, n))
    s = M.pml_steps(u, z, z, z, k, 2000)
    assert all(np.all(np.isfinite(f)) for f in s)
    assert np.max(np.abs(s[0])) < 10 * np.max(np.abs(u))


def test_host_profile_matches_oracle_bitwise():
    import paratime_b200 as B

    try:
        B.lib()
    except ImportError:
        pytest.skip("library not built")
    for n, w, h, cmax, R in [(2048, 32, 1 / 2048, 1.0, 1e-4), (256, 4, 1 / 256, 1.0, 1e-4), (100, 7, 0.013, 0.8, 1e-6)]:
        assert np.array_equal(B.damping_profile(n, w, h, cmax, R), M.damping_profile(n, w, h, cmax, R))


def _small_parareal(kind=0, N=6, K=3, nf=64, W=8):
    nc = nf // 4
    hf, hc = 1 / nf, 1 / nc
    rng = np.random.default_rng(11)
    c = 0.7 + 0.3 * rng.random((nf, nf))
    cc = np.ascontiguousarray(c[::4, ::4])
    dtf, mf = hf / 8, 16
    dtc, mc = hc / 4, 2  # the same coupling interval 1/32
    kf = M.PmlCoefficients(c, hf, hf, dtf, M.damping_profile(nf, W, hf, 1.0), M.damping_profile(nf, W, hf, 1.0))
    kc = M.PmlCoefficients(cc, hc, hc, dtc, M.damping_profile(nc, W // 4, hc, 1.0),
                           M.damping_profile(nc, W // 4, hc, 1.0))
    t = P.Transfer(P.Grid((nc, nc), (hc, hc)), P.Grid((nf, nf), (hf, hf)), kind)
    u0 = _pulse(nf, w=300.0, x0=0.45, y0=0.55)
    return dict(nf=nf, nc=nc, c=c, cc=cc, dtf=dtf, mf=mf, dtc=dtc, mc=mc, kf=kf, kc=kc, t=t, u0=u0, N=N, K=K, W=W)


@pytest.mark.parametrize("kind", [0, 1])
def test_plain_parareal_oracle_exactness_and_convergence(kind):
    s = _small_parareal(kind)
    its, err = M.plain_parareal(s["u0"], np.zeros_like(s["u0"]), s["kf"], s["mf"], s["kc"], s["mc"], s["t"],
                                s["N"], s["K"])
    for k in range(s["K"]):
        assert np.all(err[k, : k + 2] == 0.0), err[k]  # slices n <= k+1 are exact (parareal.cpp exactness)
    assert np.all(np.isfinite(err))
    if kind == 0:  # plain parareal need not converge for waves (the paper's motivation); here it does
        assert np.max(err[-1]) < np.max(err[0])


def test_theta_parareal_zero_profile_is_the_periodic_theta_oracle():
    """With no layer the layered theta coupling IS the reference's theta_engine (parareal.cpp:255-350):
    oracle/pml_np.theta_parareal on a zero profile equals oracle/paratime_np.theta_parareal (pinned
    to the compiled reference in tests/test_oracle_pin.py) to the theta path's round-off floor."""
    s = _small_parareal(0, N=6, K=3, W=8)
    nf, nc = s["nf"], s["nc"]
    hf, hc = 1 / nf, 1 / nc
    z_f, z_c = np.zeros(nf), np.zeros(nc)
    kf = M.PmlCoefficients(s["c"], hf, hf, s["dtf"], z_f, z_f)
    kc = M.PmlCoefficients(s["cc"], hc, hc, s["dtc"], z_c, z_c)
    v0 = np.zeros_like(s["u0"])
    its, err, ranks = M.theta_parareal(s["u0"], v0, kf, s["mf"], kc, s["mc"], s["t"], s["N"], s["K"], s["cc"], tol=1e-4)
    sch = P.Schedule(T=s["N"] * s["dtf"] * s["mf"], dt_com=s["dtf"] * s["mf"], n=s["N"], fine_grid=s["t"].fine,
                     c_fine=s["c"], dt_fine=s["dtf"], m_fine=s["mf"], coarse_grid=s["t"].coarse, c_coarse=s["cc"],
                     dt_coarse=s["dtc"], m_coarse=s["mc"])
    run = P.theta_parareal((s["u0"], v0), sch, s["t"], s["K"], tol=1e-4)
    for k in range(s["K"]):
        assert run.iterations[k + 1].rank == ranks[k]
        for n in range(s["N"] + 1):
            want = np.concatenate([run.iterations[k + 1].states[n][0].ravel(), run.iterations[k + 1].states[n][1].ravel()])
            got = np.concatenate([its[k][n][0].ravel(), its[k][n][1].ravel()])
            assert np.linalg.norm(got - want) <= 1e-10 * max(np.linalg.norm(want), 1e-300), (k, n)
            assert not its[k][n][2].any() and not its[k][n][3].any()


def test_theta_parareal_layer_exactness_and_stability():
    """With the layer: slices n <= k+1 are exact after iteration k (the parareal exactness property),
    and where plain parareal's iterates grow the theta coupling keeps them bounded."""
    s = _small_parareal(0, N=8, K=4, W=8)
    v0 = np.zeros_like(s["u0"])
    _, et, ranks = M.theta_parareal(s["u0"], v0, s["kf"], s["mf"], s["kc"], s["mc"], s["t"], s["N"], s["K"], s["cc"])
    for k in range(s["K"]):
        assert np.all(et[k, : k + 2] == 0.0), et[k]
    assert np.all(np.isfinite(et)) and all(r > 0 for r in ranks)
    assert list(ranks) == sorted(ranks)  # the corrector accumulates snapshots
