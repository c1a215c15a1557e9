"""Known-answer checks restated from the reference's doctest suites.

Each function takes an implementation (tests/impls.py) and asserts the property the
cited reference test asserts, with the same tolerance.  They run on the numpy oracle
(CPU suite) and on the CUDA path (``-m gpu``).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from tests.impls import Diverged, InvalidArgument

FOURIER, LINEAR = 0, 1


def unit(g):
    return np.ones(g.shape)


def rel_l2(a, b):
    """test_util.hpp:75-83"""
    a, b = np.ravel(a), np.ravel(b)
    d = float(np.sum((a - b) ** 2))
    r = float(np.sum(b * b))
    return math.sqrt(d / r) if r > 0 else math.sqrt(d)


def verlet_mode_matrix(mu, dt):
    """test_propagator.cpp:21-25"""
    k = mu * dt * dt
    return (1.0 - 0.5 * k, dt, -mu * dt * (1.0 - 0.25 * k), 1.0 - 0.5 * k)


def smooth_field(g, rng, n_modes=8):
    """test_util.hpp:22-53 (trigonometric, every mode strictly below Nyquist)"""
    if g.dim == 1:
        n = g.n[0]
        x = np.arange(n) / n
        f = np.zeros(n)
        for _ in range(n_modes):
            k = 2 * math.pi * rng.integers(0, n // 2)
            a, b = rng.uniform(-1, 1, 2)
            f += a * np.cos(k * x) + b * np.sin(k * x)
        return f
    ny, nx = g.shape
    y = (np.arange(ny) / ny)[:, None]
    x = (np.arange(nx) / nx)[None, :]
    f = np.zeros(g.shape)
    for _ in range(n_modes):
        ky = 2 * math.pi * rng.integers(0, ny // 2)
        kx = 2 * math.pi * rng.integers(0, nx // 2)
        a, b = rng.uniform(-1, 1, 2)
        f += a * np.cos(ky * y + kx * x) + b * np.sin(ky * y + kx * x)
    return f


# ------------------------------------------------------------ test_propagator.cpp


def config_enforces_cfl(impl):
    """test_propagator.cpp:30-39"""
    g = impl.grid((50,), (0.01,))
    impl.check_config(g, unit(g), 0.01, 1)
    with pytest.raises(InvalidArgument):
        impl.check_config(g, unit(g), 0.0101, 1)
    g2 = impl.grid((10, 10), (0.1, 0.1))
    impl.check_config(g2, unit(g2), 0.1 / math.sqrt(2.0), 1)
    with pytest.raises(InvalidArgument):
        impl.check_config(g2, unit(g2), 0.09, 1)
    with pytest.raises(InvalidArgument):
        impl.check_config(g, unit(g), -0.001, 1)
    with pytest.raises(InvalidArgument):
        impl.check_config(g, unit(g), 0.001, 0)


def laplacian_known_answers(impl):
    """test_propagator.cpp:41-64"""
    g = impl.grid((32,), (0.25,))
    assert np.max(np.abs(impl.laplacian(np.full(32, 4.2), g))) == 0.0
    delta = np.zeros(32)
    delta[0] = 1.0
    ld = impl.laplacian(delta, g)
    ih2 = 1.0 / (0.25 * 0.25)
    assert ld[0] == pytest.approx(-2.0 * ih2)
    assert ld[1] == pytest.approx(ih2) and ld[31] == pytest.approx(ih2)
    assert np.all(ld[2:31] == 0.0)
    gm = impl.grid((64,), (1.0 / 64,))
    xi = 2.0 * math.pi * 3.0
    mode = np.sin(xi * np.arange(64) / 64.0)
    h = 1.0 / 64
    eig = -(2.0 - 2.0 * math.cos(xi * h)) / (h * h)
    lm = impl.laplacian(mode, gm)
    np.testing.assert_allclose(lm, eig * mode, rtol=1e-10, atol=1e-10 * abs(eig))


def laplacian_2d_sum(impl):
    """test_propagator.cpp:66-82"""
    g = impl.grid((8, 16), (0.5, 0.25))
    f = np.random.default_rng(3).uniform(-1, 1, (8, 16))
    lap = impl.laplacian(f, g)
    at = lambda y, x: f[y % 8, x % 16]
    for iy in range(8):
        for ix in range(16):
            expect = ((at(iy, ix + 1) - 2.0 * at(iy, ix) + at(iy, ix - 1)) / (0.25 * 0.25)
                      + (at(iy + 1, ix) - 2.0 * at(iy, ix) + at(iy - 1, ix)) / (0.5 * 0.5))
            assert lap[iy, ix] == pytest.approx(expect, rel=1e-12, abs=1e-12)


def step_single_mode(impl):
    """test_propagator.cpp:84-112"""
    g = impl.grid((100,), (0.01,))
    dt = 0.005
    z = impl.propagate(np.zeros(100), np.zeros(100), unit(g), g, dt, 1)
    assert np.max(np.abs(z[0])) == 0.0
    xi, h = 2.0 * math.pi * 4.0, 0.01
    mu = (2.0 - 2.0 * math.cos(xi * h)) / (h * h)
    M = verlet_mode_matrix(mu, dt)
    assert M[0] * M[3] - M[1] * M[2] == pytest.approx(1.0, rel=1e-14)
    assert abs(M[0] + M[3]) <= 2.0
    x = np.arange(100) * h
    a0, b0 = 0.7, -0.3
    out = impl.propagate(a0 * np.cos(xi * x), b0 * np.cos(xi * x), unit(g), g, dt, 1)
    a1 = M[0] * a0 + M[1] * b0
    b1 = M[2] * a0 + M[3] * b0
    np.testing.assert_allclose(out[0], a1 * np.cos(xi * x), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(out[1], b1 * np.cos(xi * x), rtol=1e-12, atol=1e-12)


def second_order_in_time(impl):
    """test_propagator.cpp:114-133 (and acceptance.cpp:384-408)"""
    g = impl.grid((64,), (1.0 / 64,))
    init = np.cos(2.0 * math.pi * np.arange(64) / 64.0)
    T, dt0 = 0.5, 1.0 / 256.0

    def run(dt):
        return impl.propagate(init, np.zeros(64), unit(g), g, dt, int(round(T / dt)))

    ref = run(dt0 / 64.0)
    err = [rel_l2(run(dt0 / (1 << l))[0], ref[0]) for l in range(3)]
    slope = 0.5 * (math.log2(err[0] / err[1]) + math.log2(err[1] / err[2]))
    assert slope == pytest.approx(2.0, rel=0.05)


def repeated_step_bitwise(impl):
    """test_propagator.cpp:135-149"""
    rng = np.random.default_rng(5)
    g = impl.grid((40,), (0.025,))
    u0, v0 = smooth_field(g, rng), smooth_field(g, rng)
    manual = (u0, v0)
    for _ in range(8):
        manual = impl.propagate(manual[0], manual[1], unit(g), g, 0.01, 1)
    out = impl.propagate(u0, v0, unit(g), g, 0.01, 8)
    out2 = impl.propagate(u0, v0, unit(g), g, 0.01, 8)
    return manual, out, out2


def standing_wave(impl):
    """test_propagator.cpp:151-172"""
    g = impl.grid((100,), (0.01,))
    u = np.cos(2.0 * math.pi * np.arange(100) / 100.0)
    out = impl.propagate(u, np.zeros(100), unit(g), g, 0.005, 200)
    mu = (2.0 - 2.0 * math.cos(2.0 * math.pi * 0.01)) / (0.01 * 0.01)
    M = verlet_mode_matrix(mu, 0.005)
    a, b = 1.0, 0.0
    for _ in range(200):
        a, b = M[0] * a + M[1] * b, M[2] * a + M[3] * b
    np.testing.assert_allclose(out[0], a * u, rtol=1e-10, atol=1e-10)
    assert abs(a - 1.0) < 5e-3


def linearity(impl):
    """test_propagator.cpp:174-185"""
    rng = np.random.default_rng(9)
    g = impl.grid((48,), (1.0 / 48,))
    s1 = rng.uniform(-1, 1, (2, 48))
    s2 = rng.uniform(-1, 1, (2, 48))
    al, be = 1.7, -0.6
    lhs = impl.propagate(al * s1[0] + be * s2[0], al * s1[1] + be * s2[1], unit(g), g, 0.01, 25)
    p1 = impl.propagate(s1[0], s1[1], unit(g), g, 0.01, 25)
    p2 = impl.propagate(s2[0], s2[1], unit(g), g, 0.01, 25)
    assert rel_l2(lhs[0], al * p1[0] + be * p2[0]) <= 1e-12
    assert rel_l2(lhs[1], al * p1[1] + be * p2[1]) <= 1e-12


def reversibility(impl):
    """test_propagator.cpp:187-198"""
    rng = np.random.default_rng(15)
    g = impl.grid((64,), (1.0 / 64,))
    u0, v0 = smooth_field(g, rng), smooth_field(g, rng)
    f = impl.propagate(u0, v0, unit(g), g, 0.008, 50)
    b = impl.propagate(f[0], -f[1], unit(g), g, 0.008, 50)
    assert rel_l2(b[0], u0) <= 1e-10
    assert rel_l2(-b[1], v0) <= 1e-10


def energy_drift(impl):
    """test_propagator.cpp:200-226"""
    g = impl.grid((100,), (0.01,))
    x = -0.5 + np.arange(100) * 0.01
    s = (np.cos(10.0 * math.pi * x) * np.exp(-100.0 * x * x), np.zeros(100))

    def scheme_energy(w):
        lap = impl.laplacian(w[0], g)
        return 0.5 * float(np.sum(-w[0] * lap + w[1] * w[1])) * 0.01

    e0 = scheme_energy(s)
    emax = e0
    for _ in range(100):
        s = impl.propagate(s[0], s[1], unit(g), g, 0.00025, 200)
        e = scheme_energy(s)
        emax = max(emax, e)
        assert abs(e - e0) / e0 <= 1e-3
    assert emax / e0 <= 1.01


def divergence_reported(impl):
    """test_propagator.cpp:251-257"""
    g = impl.grid((16,), (0.0625,))
    bad = np.zeros(16)
    bad[3] = math.inf
    with pytest.raises(Diverged):
        impl.propagate(bad, np.zeros(16), unit(g), g, 0.01, 4)


# ------------------------------------------------------------ test_field_core.cpp


def grid_invariants(impl):
    """test_field_core.cpp:10-20"""
    for n, h in (((3,), (0.1,)), ((10,), (0.0,)), ((10,), (-1.0,)), ((10, 10, 10), (1.0, 1.0, 1.0))):
        with pytest.raises(InvalidArgument):
            impl.grid(n, h)


def transfer_rejects_non_nested(impl):
    """test_field_core.cpp:22-31"""
    coarse = impl.grid((10,), (0.1,))
    with pytest.raises(InvalidArgument):
        impl.transfer(coarse, impl.grid((25,), (0.04,)), LINEAR)
    with pytest.raises(InvalidArgument):
        impl.transfer(coarse, impl.grid((20,), (0.1,)), LINEAR)
    impl.transfer(coarse, impl.grid((20,), (0.05,)), LINEAR)


def restriction_pointwise(impl):
    """test_field_core.cpp:33-46"""
    coarse, fine = impl.grid((10,), (0.1,)), impl.grid((100,), (0.01,))
    t = impl.transfer(coarse, fine, FOURIER)
    assert np.all(impl.restrict(np.ones(100), t) == 1.0)
    sine = np.sin(2.0 * math.pi * np.arange(100) / 100.0)
    r = impl.restrict(sine, t)
    assert np.all(r == sine[::10])


def fourier_band_limited(impl):
    """test_field_core.cpp:48-56"""
    t = impl.transfer(impl.grid((16,), (1.0 / 16,)), impl.grid((64,), (1.0 / 64,)), FOURIER)
    out = impl.interpolate(np.cos(2.0 * math.pi * np.arange(16) / 16.0), t)
    np.testing.assert_allclose(out, np.cos(2.0 * math.pi * np.arange(64) / 64.0), rtol=1e-12, atol=1e-12)


def linear_constants_monotone(impl):
    """test_field_core.cpp:58-75"""
    t = impl.transfer(impl.grid((8,), (0.125,)), impl.grid((32,), (0.125 / 4,)), LINEAR)
    assert np.all(impl.interpolate(np.full(8, 3.25), t) == 3.25)
    u = np.random.default_rng(7).uniform(-1, 1, 8)
    out = impl.interpolate(u, t)
    for q in range(8):
        lo, hi = min(u[q], u[(q + 1) % 8]), max(u[q], u[(q + 1) % 8])
        for r in range(4):
            assert lo - 1e-15 <= out[4 * q + r] <= hi + 1e-15


def restrict_interpolate_identity(impl):
    """test_field_core.cpp:77-101 (1D and 2D, both kinds)"""
    rng = np.random.default_rng(11)
    for kind in (FOURIER, LINEAR):
        t = impl.transfer(impl.grid((20,), (0.05,)), impl.grid((100,), (0.01,)), kind)
        for _ in range(10):
            u = rng.uniform(-1, 1, 20)
            back = impl.restrict(impl.interpolate(u, t), t)
            assert np.max(np.abs(back - u)) <= 1e-12 * np.max(np.abs(u))
        t2 = impl.transfer(impl.grid((6, 10), (0.25, 0.1)), impl.grid((18, 30), (0.25 / 3, 0.1 / 3)), kind)
        for _ in range(6):
            u = rng.uniform(-1, 1, (6, 10))
            back = impl.restrict(impl.interpolate(u, t2), t2)
            assert np.max(np.abs(back - u)) <= 1e-12 * np.max(np.abs(u))


def fourier_preserves_mean(impl):
    """test_field_core.cpp:103-115"""
    t = impl.transfer(impl.grid((14,), (1.0 / 14,)), impl.grid((70,), (1.0 / 70,)), FOURIER)
    u = np.random.default_rng(17).uniform(-1, 1, 14)
    out = impl.interpolate(u, t)
    mc, mf = float(np.sum(u)) / 14.0, float(np.sum(out)) / 70.0
    assert abs(mf - mc) <= 1e-12 * max(1.0, abs(mc))


PROPAGATOR_KATS = [config_enforces_cfl, laplacian_known_answers, laplacian_2d_sum, step_single_mode,
                   second_order_in_time, standing_wave, linearity, reversibility, energy_drift,
                   divergence_reported]
TRANSFER_KATS = [grid_invariants, transfer_rejects_non_nested, restriction_pointwise, fourier_band_limited,
                 linear_constants_monotone, restrict_interpolate_identity, fourier_preserves_mean]


# ------------------------------------------------------------ test_energy_map.cpp

FD_SCHEMES = (0, 1, 2, 3)
SPECTRAL = 4


def components_constant_displacement(impl):
    """test_energy_map.cpp:50-64"""
    g = impl.grid((40,), (0.025,))
    c = np.full(40, 2.0)
    for scheme in (0, SPECTRAL):
        st, mean = impl.components(np.full(40, 5.0), c.copy(), c, g, scheme)
        assert np.max(np.abs(st[:40])) <= 1e-12
        assert np.max(np.abs(st[40:] - 1.0)) <= 1e-15
        assert mean == pytest.approx(200.0)


def spectral_gradient_exact(impl):
    """test_energy_map.cpp:66-76 (through the gradient block of Lambda)"""
    g = impl.grid((50,), (0.02,))
    x = np.arange(50) * 0.02
    u = np.sin(2 * math.pi * x)
    du = 2 * math.pi * np.cos(2 * math.pi * x)
    st, _ = impl.components(u, np.zeros(50), np.ones(50), g, SPECTRAL)
    assert np.max(np.abs(st[:50] - du)) <= 1e-12 * np.max(np.abs(du))


def fd_gradients_match_stencil(impl):
    """test_energy_map.cpp:78-92"""
    from oracle.paratime_np import STENCILS

    g = impl.grid((36,), (1.0 / 36,))
    u = np.random.default_rng(21).uniform(-1, 1, 36)
    for scheme in FD_SCHEMES:
        beta = STENCILS[scheme]
        st, _ = impl.components(u, np.zeros(36), np.ones(36), g, scheme)
        for i in range(36):
            acc = sum(b * (u[(i + j) % 36] - u[(i - j) % 36]) for j, b in enumerate(beta, start=1))
            assert st[i] == pytest.approx(acc * 36.0, rel=1e-12, abs=1e-12)


def reconstruction_inverts_spectral(impl):
    """test_energy_map.cpp:94-107 (1D 64 and 2D 12x20)"""
    rng = np.random.default_rng(33)
    for g in (impl.grid((64,), (1.0 / 64,)), impl.grid((12, 20), (1.0 / 12, 1.0 / 20))):
        c = np.ones(g.shape)
        for _ in range(5):
            u, v = smooth_field(g, rng), smooth_field(g, rng)
            st, mean = impl.components(u, v, c, g, SPECTRAL)
            bu, bv = impl.reconstruct(st, mean, c, g)
            assert rel_l2(bu, u) <= 1e-12 and rel_l2(bv, v) <= 1e-12


def fd2_reconstruction_sinc(impl):
    """test_energy_map.cpp:109-127"""
    g = impl.grid((32,), (1.0 / 32,))
    c = np.ones(32)
    h = 1.0 / 32
    for k in range(1, 16):
        xi = 2 * math.pi * k
        sinc = math.sin(xi * h) / (xi * h)
        u = np.cos(xi * np.arange(32) * h) + 0.5 * np.sin(xi * np.arange(32) * h)
        st, mean = impl.components(u, np.zeros(32), c, g, 0)
        bu, _ = impl.reconstruct(st, mean, c, g)
        np.testing.assert_allclose(bu, sinc * u, rtol=1e-12, atol=1e-12)


def zero_gradients_reconstruct_mean(impl):
    """test_energy_map.cpp:129-137"""
    g = impl.grid((25,), (0.04,))
    st = np.zeros(50)
    bu, bv = impl.reconstruct(st, 5.0, np.ones(25), g)
    assert np.max(np.abs(bu - 0.2)) <= 1e-14
    assert np.max(np.abs(bv)) == 0.0


def energy_closed_forms(impl):
    """test_energy_map.cpp:139-152"""
    g = impl.grid((80,), (0.0125,))
    c = np.full(80, 3.0)
    assert impl.energy(np.zeros(80), np.zeros(80), c, g, 0) == 0.0
    assert impl.energy(np.zeros(80), c.copy(), c, g, 0) == pytest.approx(0.5 * 80 * 0.0125)
    g2 = impl.grid((8, 10), (0.5, 0.2))
    c2 = np.full((8, 10), 1.7)
    assert impl.energy(np.zeros((8, 10)), c2.copy(), c2, g2, 1) == pytest.approx(0.5 * 80 * 0.1)


def energy_error_direct(impl):
    """test_energy_map.cpp:176-199"""
    rng = np.random.default_rng(55)
    g = impl.grid((44,), (1.0 / 44,))
    c = np.ones(44)
    a = (rng.uniform(-1, 1, 44), rng.uniform(-1, 1, 44))
    b = (rng.uniform(-1, 1, 44), rng.uniform(-1, 1, 44))
    assert impl.energy_error(b, b, c, g, 1) == 0.0
    assert impl.energy_error((2 * b[0], 2 * b[1]), b, c, g, 1) == pytest.approx(1.0)
    expect = math.sqrt(impl.energy(a[0] - b[0], a[1] - b[1], c, g, 1) / impl.energy(b[0], b[1], c, g, 1))
    assert impl.energy_error(a, b, c, g, 1) == pytest.approx(expect)
    with pytest.raises(ZeroDivisionError):
        impl.energy_error(a, (np.zeros(44), np.zeros(44)), c, g, 1)


def reconstruction_never_amplifies(impl):
    """test_energy_map.cpp:201-219"""
    rng = np.random.default_rng(61)
    for g in (impl.grid((40,), (0.025,)), impl.grid((10, 14), (0.1, 1.0 / 14))):
        c = np.ones(g.shape)
        for _ in range(3):
            u, v = rng.uniform(-1, 1, g.shape), rng.uniform(-1, 1, g.shape)
            for scheme in FD_SCHEMES + (SPECTRAL,):
                st, mean = impl.components(u, v, c, g, scheme)
                bu, bv = impl.reconstruct(st, mean, c, g)
                e_comp = 0.5 * float(np.sum(st * st)) * float(np.prod(g.h))
                assert impl.energy(bu, bv, c, g, scheme) <= e_comp * (1.0 + 1e-12)


ENERGY_KATS = [components_constant_displacement, spectral_gradient_exact, fd_gradients_match_stencil,
               reconstruction_inverts_spectral, fd2_reconstruction_sinc, zero_gradients_reconstruct_mean,
               energy_closed_forms, energy_error_direct, reconstruction_never_amplifies]


# ------------------------------------------------------------ test_procrustes.cpp / acceptance.cpp


def _haar(n, rng):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def _defect(m):
    return float(np.max(np.abs(m.T @ m - np.eye(m.shape[1])))) if m.shape[1] else 0.0


def solve_aligned_identity(impl):
    """test_procrustes.cpp:46-53"""
    G = np.random.default_rng(101).standard_normal((12, 4))
    c = impl.procrustes_solve(G, G, 1e-14)
    assert np.linalg.norm(G - c.X @ (c.Y.T @ G)) <= 1e-10 * np.linalg.norm(G)
    assert _defect(c.X) <= 1e-12 and _defect(c.Y) <= 1e-12


def solve_planted_rotation(impl):
    """test_procrustes.cpp:55-68 (wide block through the update path)"""
    rng = np.random.default_rng(103)
    al = 0.41
    rot = np.array([[math.cos(al), -math.sin(al)], [math.sin(al), math.cos(al)]])
    G = rng.standard_normal((2, 3))
    F = rot @ G
    c = impl.update_svd(None, F, G, 1e-14)
    assert c.rank == 2
    omega = c.X @ c.Y.T
    assert np.max(np.abs(omega - rot)) <= 1e-12
    assert np.linalg.norm(F - omega @ G) <= 1e-12 * np.linalg.norm(F)


def solve_matches_dense_oracle(impl):
    """test_procrustes.cpp:70-94 and acceptance criterion 2"""
    rng = np.random.default_rng(107)
    for _ in range(10):
        F = rng.standard_normal((8, 3))
        G = rng.standard_normal((8, 3))
        c = impl.procrustes_solve(F, G, 1e-15)
        res = np.linalg.norm(F - c.X @ (c.Y.T @ G))
        U, s, Vt = np.linalg.svd(F @ G.T)
        res_full = np.linalg.norm(F - (U @ Vt) @ G)
        assert res == pytest.approx(res_full, rel=1e-10)
        ident = np.sum(F * F) + np.sum(G * G) - 2.0 * np.sum(c.S)
        assert res * res == pytest.approx(ident, rel=1e-10)
        for _ in range(20):
            assert res <= np.linalg.norm(F - _haar(8, rng) @ G) + 1e-10


def zero_data_annihilates(impl):
    """test_procrustes.cpp:96-103"""
    Z = np.zeros((10, 3))
    c = impl.procrustes_solve(Z, Z, 1e-12)
    assert c.rank == 0
    out = impl.apply(c, np.ones(10))
    assert np.linalg.norm(out) == 0.0


def solve_validates(impl):
    """test_procrustes.cpp:105-115"""
    rng = np.random.default_rng(109)
    F = rng.standard_normal((6, 2))
    for args in ((F, rng.standard_normal((6, 3)), 1e-12), (rng.standard_normal((2, 6)), rng.standard_normal((2, 6)), 1e-12),
                 (F, F, 0.0), (F, F, 1.0)):
        with pytest.raises(InvalidArgument):
            impl.procrustes_solve(*args)
    with pytest.raises(InvalidArgument):
        impl.update_svd(None, F, F, -1.0)


def update_on_empty_equals_solve(impl):
    """test_procrustes.cpp:117-126"""
    rng = np.random.default_rng(113)
    F, G = rng.standard_normal((10, 4)), rng.standard_normal((10, 4))
    a = impl.procrustes_solve(F, G, 1e-13)
    b = impl.update_svd(None, F, G, 1e-13)
    assert np.max(np.abs(a.S - b.S)) <= 1e-12
    ra = a.X @ np.diag(a.S) @ a.Y.T
    rb = b.X @ np.diag(b.S) @ b.Y.T
    assert np.linalg.norm(ra - rb) <= 1e-10 * np.linalg.norm(ra)
    assert np.max(np.abs(a.X - b.X)) <= 1e-10


def chained_updates_match_dense(impl):
    """test_procrustes.cpp:128-143 and acceptance criterion 3"""
    rng = np.random.default_rng(127)
    for _ in range(5):
        c = None
        direct = np.zeros((16, 16))
        for _ in range(4):
            F, G = rng.standard_normal((16, 3)), rng.standard_normal((16, 3))
            direct += F @ G.T
            c = impl.update_svd(c, F, G, 1e-15)
            assert _defect(c.X) <= 1e-12 and _defect(c.Y) <= 1e-12
        rec = c.X @ np.diag(c.S) @ c.Y.T
        assert np.linalg.norm(rec - direct) <= 1e-10 * np.linalg.norm(direct)


def zero_block_update_unchanged(impl):
    """test_procrustes.cpp:145-153"""
    rng = np.random.default_rng(131)
    F, G = rng.standard_normal((9, 3)), rng.standard_normal((9, 3))
    c = impl.procrustes_solve(F, G, 1e-13)
    after = impl.update_svd(c, np.zeros((9, 2)), np.zeros((9, 2)), 1e-13)
    rc = c.X @ np.diag(c.S) @ c.Y.T
    ra = after.X @ np.diag(after.S) @ after.Y.T
    assert np.linalg.norm(ra - rc) <= 1e-12 * np.linalg.norm(rc)


def rank_monotone_in_tol(impl):
    """test_procrustes.cpp:155-165"""
    rng = np.random.default_rng(137)
    F, G = rng.standard_normal((20, 6)), rng.standard_normal((20, 6))
    last = 7
    for tol in (1e-15, 1e-6, 1e-2, 0.2, 0.9):
        c = impl.procrustes_solve(F, G, tol)
        assert c.rank <= last
        last = c.rank


def apply_partial_isometry(impl):
    """test_procrustes.cpp:167-193"""
    rng = np.random.default_rng(139)
    zero = impl.procrustes_solve(np.zeros((24, 2)), np.zeros((24, 2)), 1e-12)
    v = rng.uniform(-1, 1, 24)
    assert np.max(np.abs(impl.apply(zero, v))) == 0.0
    F, G = rng.standard_normal((24, 5)), rng.standard_normal((24, 5))
    pc = impl.procrustes_solve(F, G, 1e-13)
    for _ in range(10):
        v = rng.standard_normal(24)
        assert np.linalg.norm(impl.apply(pc, v)) <= np.linalg.norm(v) * (1 + 1e-12)
    aligned = impl.procrustes_solve(G, G, 1e-14)
    inr = G @ rng.standard_normal(5)
    assert np.linalg.norm(impl.apply(aligned, inr) - inr) <= 1e-10 * np.linalg.norm(inr)


def drop_leading_removes_largest(impl):
    """test_procrustes.cpp:195-207"""
    rng = np.random.default_rng(149)
    F, G = rng.standard_normal((15, 5)), rng.standard_normal((15, 5))
    c = impl.procrustes_solve(F, G, 1e-15)
    d = impl.drop_leading(c, 2)
    assert d.rank == c.rank - 2
    assert d.S[0] == c.S[2]
    assert impl.relative_residual(d, F, G) > impl.relative_residual(c, F, G)
    assert impl.drop_leading(c, c.rank + 3).rank == 0


PROCRUSTES_KATS = [solve_aligned_identity, solve_planted_rotation, solve_matches_dense_oracle, zero_data_annihilates,
                   solve_validates, update_on_empty_equals_solve, chained_updates_match_dense,
                   zero_block_update_unchanged, rank_monotone_in_tol, apply_partial_isometry,
                   drop_leading_removes_largest]
