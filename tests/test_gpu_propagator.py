"""K1 parity on the B200: every kernel family against the reference arithmetic.

EXACT mode must be bitwise equal to the oracle (itself bitwise equal to the
reference's propagator.cpp, see tests/test_oracle_pin.py); FAST mode must agree
within 1e-12 relative L2 over [u; udot] (BASELINE.json north_star)."""
import math

import numpy as np
import pytest

from oracle import paratime_np as P
from tests import kat

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-12  # relative L2 over [u; udot], north_star


@pytest.fixture(scope="module")
def impls():
    from tests.impls import CudaImpl
    import paratime_b200 as B

    return {"fast": CudaImpl(B.FAST), "exact": CudaImpl(B.EXACT)}


CASES = [
    # (grid n, h, steps, batch)  -> kernel family
    (((50,), (0.02,)), 9, 3),            # small 1D
    (((100,), (0.01,)), 64, 2),          # small 1D
    (((4096,), (1 / 4096,)), 5, 2),      # small 1D, 4 pts/thread
    (((5000,), (1 / 5000,)), 7, 2),      # streaming 1D
    (((8, 16), (0.5, 0.25)), 13, 3),     # small 2D
    (((12, 20), (1 / 12, 0.05)), 8, 2),  # small 2D
    (((64, 64), (1 / 64, 1 / 64)), 64, 2),
    (((65, 70), (1 / 65, 1 / 70)), 17, 2),     # wavefront, passes 8+8+1
    (((128, 128), (1 / 128, 1 / 128)), 64, 3),  # cfg1 fine grid
    (((37, 1030), (1 / 37, 1 / 1030)), 11, 2),  # several strips, tiny ny
    (((256, 256), (1 / 256, 1 / 256)), 64, 2),  # cfg2 fine grid
    (((200, 96), (1 / 200, 1 / 96)), 3, 1),
    (((64, 128), (1 / 64, 1 / 128)), 21, 3),    # k_cluster, cluster of 2
    (((256, 128), (1 / 256, 1 / 128)), 10, 2),  # k_cluster, cluster of 8
    (((32, 512), (1 / 32, 1 / 512)), 9, 2),     # k_cluster, cluster of 4, 4 chunks per row
    (((64, 192), (1 / 64, 1 / 192)), 19, 2),    # k_wave2 full-row strip (W = 96), passes 8+8+2+1
    (((40, 384), (1 / 40, 1 / 384)), 8, 3),     # k_wave2 full-row strip (W = 192)
]


def _inputs(grid, batch, seed):
    rng = np.random.default_rng(seed)
    shape = (batch,) + grid.shape
    u = rng.uniform(-1, 1, shape)
    v = rng.uniform(-1, 1, shape)
    c = 0.5 + 0.5 * rng.random(grid.shape)
    dt = 0.9 * min(grid.h) / (math.sqrt(grid.dim) * float(c.max()))
    return u, v, c, dt


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0][0])) + f"-m{c[1]}-b{c[2]}")
def test_exact_mode_bitwise_equals_reference(impls, case):
    (n, h), steps, batch = case
    g = P.Grid(n, h)
    u, v, c, dt = _inputs(g, batch, 1)
    ref = P.verlet_steps(u, v, c, g, dt, steps)
    got = impls["exact"].propagate_batch(u, v, c, g, dt, steps)
    assert np.array_equal(got[0], ref[0]), f"u max diff {np.max(np.abs(got[0]-ref[0]))}"
    assert np.array_equal(got[1], ref[1]), f"udot max diff {np.max(np.abs(got[1]-ref[1]))}"


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0][0])) + f"-m{c[1]}-b{c[2]}")
def test_fast_mode_within_1e12(impls, case):
    (n, h), steps, batch = case
    g = P.Grid(n, h)
    u, v, c, dt = _inputs(g, batch, 2)
    ref = P.verlet_steps(u, v, c, g, dt, steps)
    got = impls["fast"].propagate_batch(u, v, c, g, dt, steps)
    for b in range(batch):
        num = np.concatenate([got[0][b].ravel(), got[1][b].ravel()])
        den = np.concatenate([ref[0][b].ravel(), ref[1][b].ravel()])
        assert kat.rel_l2(num, den) <= FAST_TOL


def test_gaussian_pulse_config1_slice_parity(impls):
    """cfg1 fine propagator (128^2, dt = dx/8, m_F = 64) on the radial pulse."""
    n = 128
    g = P.Grid((n, n), (1 / n, 1 / n))
    y, x = np.meshgrid(np.arange(n) / n, np.arange(n) / n, indexing="ij")
    u = np.exp(-400 * ((x - 0.5) ** 2 + (y - 0.5) ** 2))[None]
    v = np.zeros_like(u)
    c = np.ones(g.shape)
    dt = 0.0625 / 64
    ref = P.verlet_steps(u, v, c, g, dt, 64)
    ex = impls["exact"].propagate_batch(u, v, c, g, dt, 64)
    assert np.array_equal(ex[0], ref[0]) and np.array_equal(ex[1], ref[1])
    fa = impls["fast"].propagate_batch(u, v, c, g, dt, 64)
    assert kat.rel_l2(np.concatenate([fa[0].ravel(), fa[1].ravel()]),
                      np.concatenate([ref[0].ravel(), ref[1].ravel()])) <= FAST_TOL


@pytest.mark.parametrize("mode", ["fast", "exact"])
@pytest.mark.parametrize("n", [(16,), (12, 20), (100, 90)])
def test_nonfinite_flags_per_slice(impls, mode, n):
    g = P.Grid(n, tuple(1.0 / k for k in n))
    u, v, c, dt = _inputs(g, 3, 4)
    u[1].flat[3] = math.inf
    v[2].flat[5] = math.nan
    _, _, flags = impls[mode].propagate_batch(u, v, c, g, dt, 4, flags=True)
    assert list(flags) == [0, 1, 1]


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_repeated_step_bitwise(impls, mode):
    manual, out, out2 = kat.repeated_step_bitwise(impls[mode])
    assert np.array_equal(out[0], out2[0]) and np.array_equal(out[1], out2[1])
    # both modes: a fused coupling is bitwise equal to the same number of single steps
    assert np.array_equal(manual[0], out[0]) and np.array_equal(manual[1], out[1])


@pytest.mark.parametrize("mode", ["fast", "exact"])
@pytest.mark.parametrize("check", kat.PROPAGATOR_KATS, ids=lambda f: f.__name__)
def test_reference_known_answers_on_gpu(impls, mode, check):
    check(impls[mode])


@pytest.mark.parametrize("check", kat.TRANSFER_KATS, ids=lambda f: f.__name__)
def test_transfer_known_answers_on_gpu(impls, check):
    check(impls["fast"])


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("shapes", [((32, 32), (128, 128)), ((64, 64), (256, 256)), ((6, 10), (18, 30)),
                                    ((20,), (100,)), ((12, 16), (12, 64)), ((9, 8), (27, 8)),
                                    # fine >= 256^2, power-of-two coarse axes: the warp-FFT route
                                    # (transfer.cu k_fourier_fft_x/y), odd ratios included; 64 x 96
                                    # has a non-power-of-two axis: the direct circulant passes
                                    ((128, 128), (512, 512)), ((64, 96), (512, 768)), ((256, 256), (1024, 1024)),
                                    ((256, 256), (2048, 2048)), ((32, 32), (256, 256)), ((128, 64), (384, 512)),
                                    ((64, 128), (512, 256))])
def test_transfer_parity(impls, kind, shapes):
    cs, fs = shapes
    coarse = P.Grid(cs, tuple(1.0 / k for k in cs))
    fine = P.Grid(fs, tuple(1.0 / k for k in fs))
    t_o = P.Transfer(coarse, fine, kind)
    impl = impls["fast"]
    t_g = impl.transfer(coarse, fine, kind)
    rng = np.random.default_rng(21)
    cf = rng.uniform(-1, 1, (3,) + coarse.shape)
    ff = rng.uniform(-1, 1, (3,) + fine.shape)
    assert np.array_equal(impl.restrict(ff, t_g), P.restrict_field(ff, t_o))
    got = impl.interpolate(cf, t_g)
    ref = P.interpolate_field(cf, t_o)
    if kind == 1:
        assert np.array_equal(got, ref)
    else:
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
