"""Generate golden fixtures from the reference itself (oracle/_ref = the reference's own
grid/propagator/energy_map/parareal .cpp compiled in place + restated FFT/Procrustes).

    python tests/golden/make_golden.py      # needs oracle/_ref (built from /root/reference)

The reference ships no data files; these small .npz fixtures let the CPU
suite pin the numpy oracle and the GPU suite pin the device path without /root/reference."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from oracle import refbind as R  # noqa: E402
from oracle.paratime_np import Grid  # noqa: E402

OUT = Path(__file__).resolve().parent
rng = np.random.default_rng(20261019)


def propagate_cases():
    out = {}
    g2 = Grid((24, 20), (1 / 24, 1 / 20))
    c2 = 0.5 + 0.5 * rng.random(g2.shape)
    u = rng.uniform(-1, 1, (2,) + g2.shape)
    v = rng.uniform(-1, 1, (2,) + g2.shape)
    dt = 0.9 * min(g2.h) / (np.sqrt(2) * c2.max())
    uo, vo, _ = R.propagate(u, v, c2, g2, dt, 13)
    out.update(p2_c=c2, p2_u0=u, p2_v0=v, p2_dt=dt, p2_steps=13, p2_u=uo, p2_v=vo)
    g1 = Grid((50,), (0.02,))
    u1, v1 = rng.uniform(-1, 1, 50), rng.uniform(-1, 1, 50)
    uo, vo, _ = R.propagate(u1, v1, np.ones(50), g1, 0.01, 9)
    out.update(p1_u0=u1, p1_v0=v1, p1_u=uo.reshape(50), p1_v=vo.reshape(50))
    return out


def transfer_cases():
    cg, fg = Grid((6, 10), (0.25, 0.1)), Grid((18, 30), (0.25 / 3, 0.1 / 3))
    f = rng.uniform(-1, 1, cg.shape)
    return dict(t_coarse=f, t_fourier=R.interpolate(f, cg, fg, 0), t_linear=R.interpolate(f, cg, fg, 1))


def energy_cases():
    g = Grid((12, 16), (1 / 12, 1 / 16))
    c = 0.5 + rng.random(g.shape)
    u, v = rng.uniform(-1, 1, g.shape), rng.uniform(-1, 1, g.shape)
    out = dict(e_c=c, e_u=u, e_v=v)
    for s in (0, 1, 4):
        st, mean = R.energy_components(u, v, c, g, s)
        out[f"e_stack{s}"] = st
        out[f"e_mean{s}"] = mean
        bu, bv = R.from_energy_components(st, mean, c, g)
        out[f"e_back{s}_u"], out[f"e_back{s}_v"] = bu, bv
        out[f"e_energy{s}"] = R.energy(u, v, c, g, s)
    return out


def procrustes_cases():
    out = {}
    corr = None
    for k in range(3):
        F = rng.standard_normal((48, 4))
        G = F + 0.1 * rng.standard_normal((48, 4))
        corr = R.update_svd(corr, F, G, 1e-12)
        X, S, Y = corr.factors()
        out.update({f"q_F{k}": F, f"q_G{k}": G, f"q_X{k}": X, f"q_S{k}": S, f"q_Y{k}": Y,
                    f"q_res{k}": corr.residual(F, G)})
    return out


def driver_cases():
    import workloads as W

    out = {}
    spec, cf, cc, u0, v0 = W.cfg1(tol=1e-8)
    rs = R.RunSpec()
    rs.dim = 2
    for k in range(2):
        rs.fine_n[k], rs.fine_h[k] = spec["fine_n"][k], spec["fine_h"][k]
        rs.coarse_n[k], rs.coarse_h[k] = spec["coarse_n"][k], spec["coarse_h"][k]
    for k in ("dt_fine", "m_fine", "dt_coarse", "m_coarse", "T", "dt_com", "n_couplings", "interp", "iterations",
              "variant", "scheme", "metric_scheme", "tol", "remove_leading"):
        setattr(rs, k, spec[k])
    rs.workers = 4
    r = R.parareal_run(rs, cf, cc, u0, v0, keep_states=True)
    out.update(d1_energy_err=r["energy_err"], d1_l2_err=r["l2_err"], d1_rank=r["rank"], d1_residual=r["residual"],
               d1_final=r["states"][-1, -1], d1_mid=r["states"][2, 8])
    spec_r, cf1, cc1, u1, v1 = R.build_setup("rank-tolerance", overrides="iterations=4\nT=2\ntol=1e-8")
    r1 = R.parareal_run(spec_r, cf1, cc1, u1, v1, keep_states=True)
    out.update(d2_c=cf1, d2_u0=u1, d2_energy_err=r1["energy_err"], d2_rank=r1["rank"], d2_final=r1["states"][-1, -1],
               d2_spec=np.array([spec_r.fine_n[0], spec_r.fine_h[0], spec_r.coarse_n[0], spec_r.coarse_h[0],
                                 spec_r.dt_fine, spec_r.m_fine, spec_r.dt_coarse, spec_r.m_coarse, spec_r.T,
                                 spec_r.dt_com, spec_r.n_couplings, spec_r.interp, spec_r.iterations,
                                 spec_r.variant, spec_r.scheme]))
    return out


if __name__ == "__main__":
    data = {}
    for f in (propagate_cases, transfer_cases, energy_cases, procrustes_cases, driver_cases):
        data.update(f())
    np.savez_compressed(OUT / "reference_fixtures.npz", **data)
    print("wrote", OUT / "reference_fixtures.npz", sum(v.nbytes for v in map(np.asarray, data.values())), "bytes")
