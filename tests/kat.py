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
