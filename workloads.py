"""Seeded synthetic inputs for the BASELINE.json configurations (bench + tests).

BASELINE.json lists five configs; the reference publishes no data for them (SURVEY.md
8(c)), so every field here is generated from a fixed seed (20261019 + cfg) with numpy's
PCG64 and documented in DESIGN.md.  T = 1 where BASELINE.json leaves it open (cfg 2-4).

Each cfgN() returns (spec, c_fine, c_coarse, u0, udot0) where `spec` holds the keyword
fields of the C ABI's ptb_run_spec (include/paratime_b200.h).
"""
from __future__ import annotations

import math

import numpy as np

SEED = 20261019


def _mesh(n):
    y, x = np.meshgrid(np.arange(n) / n, np.arange(n) / n, indexing="ij")
    return y, x


def _spec(nf, nc, N, K, m_f, m_c, tol, variant=1, scheme=0, interp=0, mode=0):
    dt_com = 1.0 / N
    return dict(dim=2, fine_n=(nf, nf), fine_h=(1 / nf, 1 / nf), coarse_n=(nc, nc), coarse_h=(1 / nc, 1 / nc),
                dt_fine=dt_com / m_f, m_fine=m_f, dt_coarse=dt_com / m_c, m_coarse=m_c, T=1.0, dt_com=dt_com,
                n_couplings=N, interp=interp, iterations=K, variant=variant, scheme=scheme, metric_scheme=scheme,
                tol=tol, remove_leading=0, mode=mode)


def restrict(c, r):
    return np.ascontiguousarray(c[::r, ::r])


def cfg1(tol=1e-8, **kw):
    """c = 1, 128^2 / 32^2, N = 16, K = 4, u0 = exp(-400 |x - (0.5, 0.5)|^2), udot0 = 0."""
    nf, nc = 128, 32
    y, x = _mesh(nf)
    u0 = np.exp(-400.0 * ((x - 0.5) ** 2 + (y - 0.5) ** 2))
    c = np.ones((nf, nf))
    return _spec(nf, nc, 16, 4, 64, 8, tol, **kw), c, restrict(c, 4), u0, np.zeros_like(u0)


def cfg2(tol=1e-4, **kw):
    """c = 1 - 0.25 sin(2 pi x) sin(2 pi y), 256^2 / 64^2, N = 32, K = 6, Gaussian pulse with a
    seeded centre x0 ~ U[0.3, 0.7]^2."""
    nf, nc = 256, 64
    rng = np.random.default_rng(SEED + 2)
    y0, x0 = rng.uniform(0.3, 0.7, 2)
    y, x = _mesh(nf)
    c = 1.0 - 0.25 * np.sin(2 * math.pi * x) * np.sin(2 * math.pi * y)
    u0 = np.exp(-400.0 * ((x - x0) ** 2 + (y - y0) ** 2))
    return _spec(nf, nc, 32, 6, 64, 8, tol, **kw), c, restrict(c, 4), u0, np.zeros_like(u0)


def layered_faulted(n, rng, layers=12, faults=3, cmin=0.27, cmax=1.0, noise=0.03):
    """Seeded layered-faulted medium: sorted uniform interface depths, velocities rising with
    depth in [cmin, cmax], +-3% i.i.d. uniform noise, `faults` dipping faults that offset the
    layering by 5-20 cells.  Row = depth (axis 0)."""
    depths = np.sort(rng.uniform(0, 1, layers - 1))
    vel = np.sort(rng.uniform(cmin, cmax, layers))
    vel[0], vel[-1] = cmin, cmax
    ycell = (np.arange(n) + 0.5) / n
    xcell = (np.arange(n) + 0.5) / n
    shift = np.zeros((n, n))  # depth shift (in fraction of the box) applied per cell
    for _ in range(faults):
        x_top = rng.uniform(0.2, 0.8)
        dip = rng.uniform(-0.5, 0.5)  # dx per unit depth
        offset = rng.integers(5, 21) / n
        yy, xx = np.meshgrid(ycell, xcell, indexing="ij")
        side = xx > (x_top + dip * yy)  # hanging wall
        shift += np.where(side, offset, 0.0)
    yy, _ = np.meshgrid(ycell, xcell, indexing="ij")
    layer = np.searchsorted(depths, (yy - shift) % 1.0)
    c = vel[layer]
    c *= 1.0 + noise * rng.uniform(-1, 1, (n, n))
    return c


def gaussian_smooth_periodic(c, sigma):
    """Periodic Gaussian smoothing (FFT), sigma in cells."""
    n = c.shape[0]
    k = np.fft.fftfreq(n) * 2 * math.pi
    g = np.exp(-0.5 * (sigma ** 2) * (k[:, None] ** 2 + k[None, :] ** 2))
    return np.real(np.fft.ifft2(np.fft.fft2(c) * g))


def cfg3(tol=1e-4, **kw):
    """Layered-faulted medium 512^2 / 128^2, N = 64, K = 8; coarse c = Gaussian-smoothed
    (sigma = m_s/2 = 2 fine cells) then restricted fine c; u0 = exp(-2500 |x - x0|^2) near the top."""
    nf, nc = 512, 128
    rng = np.random.default_rng(SEED + 3)
    c = layered_faulted(nf, rng)
    cc = restrict(gaussian_smooth_periodic(c, 2.0), 4)
    y, x = _mesh(nf)
    x0 = rng.uniform(0.3, 0.7)
    u0 = np.exp(-2500.0 * ((x - x0) ** 2 + (y - 0.15) ** 2))
    return _spec(nf, nc, 64, 8, 64, 8, tol, **kw), c, cc, u0, np.zeros_like(u0)


def cfg4(tol=1e-4, **kw):
    """The cfg3 generator at 2048^2 / 256^2, N = 128, K = 8, m_F = 128, m_C = 8 (m_s = 8, m_t = 16);
    coarse c = Gaussian-smoothed (sigma = m_s/2 = 4 fine cells) then restricted fine c;
    u0 = exp(-40000 |x - x0|^2) near the top.  PERIODIC: BASELINE's 32-cell absorbing layer is not
    part of the reference (no oracle), so the periodic problem is the
    parity-checkable stand-in."""
    nf, nc = 2048, 256
    rng = np.random.default_rng(SEED + 4)
    c = layered_faulted(nf, rng)
    cc = restrict(gaussian_smooth_periodic(c, 4.0), 8)
    y, x = _mesh(nf)
    x0 = rng.uniform(0.3, 0.7)
    u0 = np.exp(-40000.0 * ((x - x0) ** 2 + (y - 0.15) ** 2))
    return _spec(nf, nc, 128, 8, 128, 8, tol, **kw), c, cc, u0, np.zeros_like(u0)


def cfg4_pml(reflection=1e-4, profile=None):
    """cfg4 with BASELINE.json's 32-cell absorbing layer on all sides (fine 2048^2: 32 cells; coarse
    256^2: the same physical width, 4 cells), quadratic damping profile with amplitude
    1.5 cmax ln(1/R)/L, R = 1e-4, cmax = max fine c for both grids.  Returns
    (spec, c_fine, c_coarse, u0, udot0, (zeta_fine, zeta_coarse)); the profiles are per axis (the
    same for rows and columns).  The reference has no layer: this runs
    theta-parareal with the layer through ptb_pml_theta_run."""
    if profile is None:  # the C ABI's host profile (bitwise equal to oracle/pml_np.damping_profile)
        from paratime_b200 import damping_profile as profile
    spec, c, cc, u0, v0 = cfg4()
    nf, nc = spec["fine_n"][0], spec["coarse_n"][0]
    cmax = float(c.max())
    zf = profile(nf, 32, 1.0 / nf, cmax, reflection)
    zc = profile(nc, 4, 1.0 / nc, cmax, reflection)
    return spec, c, cc, u0, v0, (zf, zc)


def cfg5_medium(n, seed=SEED + 5):
    """c = 0.75 + 0.25 S/max|S|, S = sum of 8 sinusoids of integer wavenumbers 1..4."""
    rng = np.random.default_rng(seed)
    y, x = _mesh(n)
    s = np.zeros((n, n))
    for _ in range(8):
        ky, kx = rng.integers(1, 5, 2)
        s += rng.uniform(0.2, 1.0) * np.sin(2 * math.pi * (ky * y + kx * x) + rng.uniform(0, 2 * math.pi))
    return 0.75 + 0.25 * s / np.max(np.abs(s))


def cfg5_pulses(n, batch, seed=SEED + 50):
    """"Random Gaussian initial states": exp(-w |x - x0|^2), x0 ~ U[0,1)^2 (periodic distance),
    w ~ U[200, 2000], udot0 = 0."""
    rng = np.random.default_rng(seed)
    ax = np.arange(n) / n
    out = np.empty((batch, n, n))
    for b in range(batch):
        y0, x0 = rng.random(2)
        w = rng.uniform(200, 2000)
        dy = np.minimum(np.abs(ax - y0), 1 - np.abs(ax - y0))[:, None]
        dx = np.minimum(np.abs(ax - x0), 1 - np.abs(ax - x0))[None, :]
        out[b] = np.exp(-w * (dy * dy + dx * dx))
    return out


def cfg4_subset(n_couplings=16, iterations=2, tol=1e-4):
    """BASELINE config 4 (periodic, 2048^2 / 256^2, m_F = 128, m_C = 8) over its first
    `n_couplings` coupling intervals (T = n_couplings / 128, same dt_com and inputs): small enough
    for the CPU reference (parity tests, the CPU s/iteration sample), and 3 N_c x r = 196608 x r
    > 4M corrector entries, so the device sweep takes its large-corrector branch as the full
    config does."""
    spec, cf, cc, u0, v0 = cfg4(tol=tol)
    spec = dict(spec)
    spec["n_couplings"] = n_couplings
    spec["T"] = n_couplings * spec["dt_com"]
    spec["iterations"] = iterations
    return spec, cf, cc, u0, v0


CONFIGS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4}


def cfg5_pulse_params(batch, seed=SEED + 50):
    """(y0, x0, w) per slice for cfg5_pulses_device (same draws, same order as cfg5_pulses)."""
    rng = np.random.default_rng(seed)
    out = np.empty((batch, 3))
    for b in range(batch):
        out[b, :2] = rng.random(2)
        out[b, 2] = rng.uniform(200, 2000)
    return out


def cfg5_pulses_device(n, batch, out, seed=SEED + 50):
    """cfg5 initial states written straight into the device tensor `out` (batch, n, n), for
    batches too large to stage on the host (4096^2 x 512 slices = 69 GB per field):
    exp(-w dy^2) * exp(-w dx^2) with periodic distances.  Deterministic (same bits on every
    call), so a parity check can regenerate the inputs and hand the same slices to the
    reference."""
    import torch

    ax = torch.arange(n, dtype=torch.float64, device=out.device) / n
    for b, (y0, x0, w) in enumerate(cfg5_pulse_params(batch, seed)):
        dy = torch.minimum((ax - y0).abs(), 1 - (ax - y0).abs())
        dx = torch.minimum((ax - x0).abs(), 1 - (ax - x0).abs())
        torch.outer(torch.exp(-w * dy * dy), torch.exp(-w * dx * dx), out=out[b])
    return out
