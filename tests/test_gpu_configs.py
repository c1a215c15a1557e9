"""Parity on the BASELINE.json configurations against the reference itself (oracle/_ref).

North star acceptance: parareal iterates within 1e-10 relative energy norm of the reference
CPU implementation on the same seeded inputs.  Every case here runs the reference's own
theta_parareal (parareal.cpp:255-350, compiled verbatim; Procrustes restated on LAPACK) on the
GPU box's host cores and the device driver on the same workloads.py inputs, then compares
every iterate (k, n) with the reference's energy_error (energy_map.cpp:228-236) and l2_error
(:238-249).  tol = 1e-4 for configs 2-4: the oracle's own self-sensitivity floor there is
<= 1e-12 (profiles/r02_noise_floor.json, scripts/noise_floor.py); at tol <= 1e-10 the
theta path amplifies last-bit differences past 1e-10 (SURVEY.md addendum), so those
tolerances are reported beside the floor, not asserted.
"""
import numpy as np
import pytest

import workloads as W
from tests import configs as T

pytestmark = pytest.mark.gpu

ITERATE_TOL = 1e-10  # relative energy norm, north_star
L2_TOL = 1e-9  # l2_error of u (catches a constant offset the energy seminorm cannot see)


def _gpu(spec, cf, cc, u0, v0):
    import paratime_b200 as B

    ctx = B.Context(0)
    return B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, keep_states=True)


def _check(ref, spec, cf, cc, u0, v0):
    gpu = _gpu(spec, cf, cc, u0, v0)
    want = T.reference_run(ref, spec, cf, cc, u0, v0, keep_states=True)
    assert list(gpu["rank"]) == list(want["rank"]), (gpu["rank"], want["rank"])
    assert list(gpu["diverged"]) == list(want["diverged"])
    ee, l2 = T.iterate_distance(ref, gpu["states"], want["states"], cf, T.fine_grid(spec), spec["metric_scheme"])
    print("iterate energy distance per k", ee.max(axis=1), "l2", l2.max(axis=1))
    assert ee.max() <= ITERATE_TOL, (ee.max(axis=1), ee.argmax())
    assert l2.max() <= L2_TOL, l2.max(axis=1)
    # the per-iteration error tables against the serial fine run agree as well
    np.testing.assert_allclose(gpu["energy_err"], want["energy_err"], rtol=1e-7, atol=1e-13)
    np.testing.assert_allclose(gpu["l2_err"], want["l2_err"], rtol=1e-7, atol=1e-13)
    return gpu, want, ee


def test_config2_theta_iterates_match_reference(ref):
    """BASELINE config 2: 256^2 / 64^2, c = 1 - 0.25 sin sin, N = 32, K = 6, tol 1e-4."""
    _check(ref, *W.cfg2())


def test_config3_theta_iterates_match_reference(ref):
    """BASELINE config 3: seeded layered-faulted medium, 512^2 / 128^2, N = 64, K = 8, tol 1e-4."""
    _check(ref, *W.cfg3())


def test_config4_reduced_theta_iterates_match_reference(ref, monkeypatch):
    """BASELINE config 4 (periodic) over its first 16 couplings, K = 2: the full 2048^2 / 256^2
    schedule (m_F = 128, m_C = 8, sigma = 4 smoothing).  The sweep's large-corrector branch
    (the one the full config's 196608 x ~1000 corrector takes) is forced by lowering its
    threshold below this run's 196608 x r entries."""
    monkeypatch.setenv("PTB_FUSED_SWEEP_MAX", "1000000")
    gpu, want, ee = _check(ref, *T.reduced_cfg4())
    assert gpu["rank"][-1] * 3 * 256 * 256 > 1_000_000


def test_config1_plain_and_theta_default_tol(ref):
    """Config 1 at the reference's default truncation tol (1e-15, parareal.hpp:52) and the
    paper's 1e-13: the floor there (profiles/r02_noise_floor.json) is ~1e-11, so the device
    must stay within 1e-10 of the reference."""
    for tol in (1e-13, 1e-15):
        spec, cf, cc, u0, v0 = W.cfg1(tol=tol)
        _check(ref, spec, cf, cc, u0, v0)
