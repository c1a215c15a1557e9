"""Absorbing-layer (PML) fine propagator on the B200 against oracle/pml_np.py.

The reference has no PML: the oracle is this build's own specification,
pinned by tests/test_pml_oracle.py.  Tolerance 1e-12 relative L2 per field (fp64, FMA-contracted
kernel vs the numpy restatement); a zero profile must reproduce the periodic FAST kernels bitwise."""
import numpy as np
import pytest

from oracle import pml_np as M

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    import paratime_b200 as B

    return B.Context(0)


def _case(ny, nx, hy, hx, w, batch, seed, layer_noise=True):
    rng = np.random.default_rng(seed)
    c = 0.5 + 0.5 * rng.random((ny, nx))
    zy = M.damping_profile(ny, w, hy, 1.0, 1e-4)
    zx = M.damping_profile(nx, w, hx, 1.0, 1e-4)
    u = rng.standard_normal((batch, ny, nx))
    v = rng.standard_normal((batch, ny, nx))
    mask = (zy[:, None] > 0) | (zx[None, :] > 0)
    px = rng.standard_normal((batch, ny, nx)) * mask if layer_noise else np.zeros((batch, ny, nx))
    py = rng.standard_normal((batch, ny, nx)) * mask if layer_noise else np.zeros((batch, ny, nx))
    return c, zy, zx, (u, v, px, py)


def _rel(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


@pytest.mark.parametrize(
    "ny,nx,w,steps,batch",
    [
        (64, 64, 8, 4, 2),      # one pass
        (64, 64, 8, 9, 2),      # passes 4+4+1 (odd: result copied back from scratch)
        (96, 80, 6, 7, 3),      # partial tiles, non-square grid
        (128, 128, 16, 16, 2),  # cfg1-size grid, 4 passes
        (40, 24, 5, 5, 1),      # grid smaller than the haloed tile (multiple periodic wraps)
        (256, 192, 32, 12, 1),  # cfg4's 32-cell layer
    ],
)
def test_pml_matches_oracle(ctx, ny, nx, w, steps, batch):
    import paratime_b200 as B

    hy, hx = 1 / ny, 1 / nx
    dt = min(hy, hx) / 8
    c, zy, zx, st = _case(ny, nx, hy, hx, w, batch, seed=ny * 7 + nx)
    k = M.PmlCoefficients(c, hy, hx, dt, zy, zx)
    want = M.pml_steps(*st, k, steps)
    prop = B.PmlPropagator(ctx, B.Grid((ny, nx), (hy, hx)), c, zy, zx, dt, steps)
    t = [ctx.tensor(a) for a in st]
    flags = ctx.torch.zeros(batch, dtype=ctx.torch.int32, device="cuda:0")
    prop.propagate(*t, flags=flags)
    got = [x.cpu().numpy() for x in t]
    for name, g, r in zip(("u", "udot", "px", "py"), got, want):
        assert _rel(g, r) <= TOL, (name, _rel(g, r))
    assert not flags.cpu().numpy().any()


@pytest.mark.parametrize("n,steps", [(128, 64), (256, 8), (100, 13)])
def test_zero_profile_is_periodic_fast_bitwise(ctx, n, steps):
    import paratime_b200 as B

    h = 1 / n
    rng = np.random.default_rng(n)
    c = 0.5 + 0.5 * rng.random((n, n))
    u = rng.standard_normal((2, n, n))
    v = rng.standard_normal((2, n, n))
    g = B.Grid((n, n), (h, h))
    pml = B.PmlPropagator(ctx, g, c, np.zeros(n), np.zeros(n), h / 8, steps)
    per = B.Propagator(ctx, g, c, h / 8, steps)
    a = [ctx.tensor(u), ctx.tensor(v), ctx.tensor(np.zeros_like(u)), ctx.tensor(np.zeros_like(u))]
    b = [ctx.tensor(u), ctx.tensor(v)]
    pml.propagate(*a)
    per.propagate(*b, mode=B.FAST)
    assert np.array_equal(a[0].cpu().numpy(), b[0].cpu().numpy())
    assert np.array_equal(a[1].cpu().numpy(), b[1].cpu().numpy())


def test_fused_equals_repeated_single_steps(ctx):
    import paratime_b200 as B

    n, w, steps = 96, 12, 10
    h = 1 / n
    c, zy, zx, st = _case(n, n, h, h, w, 2, seed=5)
    prop = B.PmlPropagator(ctx, B.Grid((n, n), (h, h)), c, zy, zx, h / 8, steps)
    a = [ctx.tensor(x) for x in st]
    b = [ctx.tensor(x) for x in st]
    prop.propagate(*a)
    for _ in range(steps):
        prop.propagate(*b, steps=1)
    for x, y in zip(a, b):
        assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_nonfinite_flag(ctx):
    import paratime_b200 as B

    n = 64
    h = 1 / n
    c, zy, zx, st = _case(n, n, h, h, 8, 3, seed=9)
    st[0][1, 3, 3] = np.nan
    prop = B.PmlPropagator(ctx, B.Grid((n, n), (h, h)), c, zy, zx, h / 8, 4)
    t = [ctx.tensor(a) for a in st]
    flags = ctx.torch.zeros(3, dtype=ctx.torch.int32, device="cuda:0")
    prop.propagate(*t, flags=flags)
    assert flags.cpu().numpy().tolist() == [0, 1, 0]


def test_cfl_and_shape_errors(ctx):
    import paratime_b200 as B

    n = 32
    g = B.Grid((n, n), (1 / n, 1 / n))
    with pytest.raises(B.PtbError):
        B.PmlPropagator(ctx, g, np.ones((n, n)), np.zeros(n), np.zeros(n), 1.0 / n, 4)  # CFL
    with pytest.raises(B.PtbError):
        B.PmlPropagator(ctx, g, np.ones((n, n)), -np.ones(n), np.zeros(n), 0.1 / n, 4)  # negative damping


def test_pulse_absorbed_on_device(ctx):
    """cfg4-like: 512^2 with a 32-cell layer, constant speed; the interior energy drops once the
    pulse has crossed the layer and the run stays finite."""
    import paratime_b200 as B

    n, w = 512, 32
    h = 1 / n
    y, x = np.meshgrid(np.arange(n) / n, np.arange(n) / n, indexing="ij")
    u0 = np.exp(-2500 * ((x - 0.5) ** 2 + (y - 0.5) ** 2))
    c = np.ones((n, n))
    zs = M.damping_profile(n, w, h, 1.0, 1e-4)
    prop = B.PmlPropagator(ctx, B.Grid((n, n), (h, h)), c, zs, zs, h / 8, 4096)
    z = np.zeros((n, n))
    t = [ctx.tensor(u0), ctx.tensor(z), ctx.tensor(z), ctx.tensor(z)]
    e0 = M.interior_energy(u0, z, c, h, h, w)
    prop.propagate(*t)  # t = 1: the front has crossed the layer
    e1 = M.interior_energy(t[0].cpu().numpy(), t[1].cpu().numpy(), c, h, h, w)
    assert np.isfinite(e1) and e1 < 1e-2 * e0, e1 / e0


@pytest.mark.parametrize("kind,nf,width", [(0, 64, 8), (1, 64, 8), (0, 256, 32), (1, 256, 32)])
def test_pml_plain_parareal_matches_oracle(ctx, kind, nf, width):
    """Iterates of the device driver vs oracle/pml_np.plain_parareal (1e-10 relative per field,
    the north star's iterate tolerance) and bitwise exactness of the converged slices.  At 256^2
    with a 32-cell layer (config 4's width) the interior is covered by plain tiles (k_pml_plain)
    and the Fourier-interpolated auxiliary fields are cut back to the layer."""
    import paratime_b200 as B
    from tests.test_pml_oracle import _small_parareal

    s = _small_parareal(kind, N=5 if nf > 64 else 6, nf=nf, W=width)
    its, err = M.plain_parareal(s["u0"], np.zeros_like(s["u0"]), s["kf"], s["mf"], s["kc"], s["mc"], s["t"],
                                s["N"], s["K"])
    nf, nc, W = s["nf"], s["nc"], s["W"]
    gf, gc = B.Grid((nf, nf), (1 / nf, 1 / nf)), B.Grid((nc, nc), (1 / nc, 1 / nc))
    zf = M.damping_profile(nf, W, 1 / nf, 1.0)
    zc = M.damping_profile(nc, W // 4, 1 / nc, 1.0)
    fine = B.PmlPropagator(ctx, gf, s["c"], zf, zf, s["dtf"], s["mf"])
    coarse = B.PmlPropagator(ctx, gc, s["cc"], zc, zc, s["dtc"], s["mc"])
    tr = B.Transfer(ctx, gc, gf, kind)
    r = B.pml_parareal_run(fine, coarse, tr, s["N"], s["K"], s["u0"], np.zeros_like(s["u0"]), keep_states=True)
    assert not r["diverged"]
    last = its[-1]
    for f in range(4):
        want = np.stack([last[n][f] for n in range(s["N"] + 1)])
        got = r["states"][f]
        assert _rel(got, want) <= 1e-10, (f, _rel(got, want))
    for k in range(s["K"]):
        assert np.all(r["rel_err"][k, : k + 2] == 0.0), r["rel_err"][k]  # exact slices, bitwise
    np.testing.assert_allclose(r["rel_err"][:, s["K"] + 1:], err[:, s["K"] + 1:], rtol=1e-8)
    assert np.all(r["iteration_ms"] > 0)


def test_cxx_api_suite():
    """tests/refsuite/test_pml.cpp: the C++ drop-in extension (include/paratime/pml.hpp) in the
    reference's doctest style, built in the development container."""
    import subprocess
    from pathlib import Path

    exe = Path(__file__).resolve().parent / "refsuite" / "_bin" / "test_pml"
    if not exe.exists():
        pytest.skip(f"{exe} not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failed checks: 0" in r.stdout


@pytest.mark.parametrize("world", [2, 3])
def test_pml_parareal_sharded_equals_single_gpu(world):
    """The slice-sharded layered driver (loopback communicator: in-process ranks on cuda:0, the same
    C++ all-gather / boundary-shift code as NCCL) is bitwise equal to one GPU."""
    import threading

    import paratime_b200 as B
    from tests.test_pml_oracle import _small_parareal

    s = _small_parareal(0, N=7, K=3)
    nf, nc, W = s["nf"], s["nc"], s["W"]
    gf, gc = B.Grid((nf, nf), (1 / nf, 1 / nf)), B.Grid((nc, nc), (1 / nc, 1 / nc))
    zf = M.damping_profile(nf, W, 1 / nf, 1.0)
    zc = M.damping_profile(nc, W // 4, 1 / nc, 1.0)
    v0 = np.zeros_like(s["u0"])

    def objects(c):
        return (B.PmlPropagator(c, gf, s["c"], zf, zf, s["dtf"], s["mf"]),
                B.PmlPropagator(c, gc, s["cc"], zc, zc, s["dtc"], s["mc"]), B.Transfer(c, gc, gf, 0))

    c1 = B.Context(0)
    single = B.pml_parareal_run(*objects(c1), s["N"], s["K"], s["u0"], v0, keep_states=True)
    group = B.api.LoopbackGroup(world)
    ctxs = [B.Context(0).use_own_stream() for _ in range(world)]  # a stream per rank
    objs = [objects(c) for c in ctxs]
    comms = [group.comm(ctxs[r], r) for r in range(world)]
    out, err = [None] * world, []

    def work(r):
        try:
            out[r] = B.pml_parareal_run(*objs[r], s["N"], s["K"], s["u0"], v0, keep_states=True, comm=comms[r])
        except Exception as e:  # pragma: no cover
            err.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not err, err
    N = s["N"]
    chunk = -(-N // world)
    for r, o in enumerate(out):
        assert np.array_equal(o["rel_err"], single["rel_err"])
        a = 1 + r * chunk
        b = min(N + 1, a + chunk)
        assert np.array_equal(o["states"][:, a - 1:b], single["states"][:, a - 1:b])


@pytest.mark.parametrize("kind,nf,width", [(0, 64, 8), (1, 64, 8), (0, 256, 32)])
def test_pml_theta_parareal_matches_oracle(ctx, kind, nf, width):
    """Theta (Procrustes) parareal with the absorbing layer (ptb_pml_theta_run) vs
    oracle/pml_np.theta_parareal: corrector ranks equal, iterates within 1e-10 relative per field
    (the north star's iterate tolerance; tol 1e-4 as the periodic config tests), converged slices exact."""
    import paratime_b200 as B
    from tests.test_pml_oracle import _small_parareal

    s = _small_parareal(kind, N=5 if nf > 64 else 7, K=3, nf=nf, W=width)
    v0 = np.zeros_like(s["u0"])
    its, err, ranks = M.theta_parareal(s["u0"], v0, s["kf"], s["mf"], s["kc"], s["mc"], s["t"], s["N"], s["K"],
                                       s["cc"], tol=1e-4)
    nf, nc, W = s["nf"], s["nc"], s["W"]
    gf, gc = B.Grid((nf, nf), (1 / nf, 1 / nf)), B.Grid((nc, nc), (1 / nc, 1 / nc))
    zf = M.damping_profile(nf, W, 1 / nf, 1.0)
    zc = M.damping_profile(nc, W // 4, 1 / nc, 1.0)
    fine = B.PmlPropagator(ctx, gf, s["c"], zf, zf, s["dtf"], s["mf"])
    coarse = B.PmlPropagator(ctx, gc, s["cc"], zc, zc, s["dtc"], s["mc"])
    tr = B.Transfer(ctx, gc, gf, kind)
    r = B.pml_theta_run(fine, coarse, tr, s["N"], s["K"], s["u0"], v0, tol=1e-4, keep_states=True)
    assert not r["diverged"]
    assert list(r["rank"]) == list(ranks), (r["rank"], ranks)
    last = its[-1]
    for f in range(4):
        want = np.stack([last[n][f] for n in range(s["N"] + 1)])
        got = r["states"][f]
        assert _rel(got, want) <= 1e-10, (f, _rel(got, want))
    for k in range(s["K"]):  # converged slices: exact up to the sweep's round-off (corrected(old[n]) is a
        # batched product, corrected(w) a per-step one; test_gpu_path.py applies the same bound)
        assert np.all(r["rel_err"][k, : k + 2] <= 1e-12), r["rel_err"][k]
    np.testing.assert_allclose(r["rel_err"][:, s["K"] + 1:], err[:, s["K"] + 1:], rtol=1e-7)
    assert np.all(r["residual"] >= 0) and np.all(r["iteration_ms"] > 0)


@pytest.mark.parametrize("world", [2, 3])
def test_pml_theta_sharded_equals_single_gpu(world):
    """Theta with the layer, slices sharded over loopback ranks: bitwise equal to one GPU (the stage
    flags travel with the coarse payload; the corrector fit and the sweep are replicated)."""
    import threading

    import paratime_b200 as B
    from tests.test_pml_oracle import _small_parareal

    s = _small_parareal(0, N=7, K=3)
    nf, nc, W = s["nf"], s["nc"], s["W"]
    gf, gc = B.Grid((nf, nf), (1 / nf, 1 / nf)), B.Grid((nc, nc), (1 / nc, 1 / nc))
    zf = M.damping_profile(nf, W, 1 / nf, 1.0)
    zc = M.damping_profile(nc, W // 4, 1 / nc, 1.0)
    v0 = np.zeros_like(s["u0"])

    def objects(c):
        return (B.PmlPropagator(c, gf, s["c"], zf, zf, s["dtf"], s["mf"]),
                B.PmlPropagator(c, gc, s["cc"], zc, zc, s["dtc"], s["mc"]), B.Transfer(c, gc, gf, 0))

    single = B.pml_theta_run(*objects(B.Context(0)), s["N"], s["K"], s["u0"], v0, keep_states=True)
    group = B.api.LoopbackGroup(world)
    ctxs = [B.Context(0).use_own_stream() for _ in range(world)]  # a stream per rank
    objs = [objects(c) for c in ctxs]
    comms = [group.comm(ctxs[r], r) for r in range(world)]
    out, errs = [None] * world, []

    def work(r):
        try:
            out[r] = B.pml_theta_run(*objs[r], s["N"], s["K"], s["u0"], v0, keep_states=True, comm=comms[r])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    chunk = -(-s["N"] // world)
    for r, o in enumerate(out):
        assert np.array_equal(o["rel_err"], single["rel_err"])
        assert list(o["rank"]) == list(single["rank"])
        a = 1 + r * chunk
        b = min(s["N"] + 1, a + chunk)
        assert np.array_equal(o["states"][:, a - 1:b], single["states"][:, a - 1:b])


@pytest.mark.parametrize("ny,nx,w,steps,batch", [(512, 512, 32, 8, 2), (512, 512, 32, 20, 1), (640, 448, 24, 13, 3),
                                                 (448, 704, 32, 16, 2)])
def test_super_pass_equals_short_passes_bitwise(ctx, ny, nx, w, steps, batch, monkeypatch):
    """Super-pass (the interior advances 8 steps in one wavefront launch; the bands run two 4-step
    passes, the first on wider bands into a third buffer set) against 4-step passes only: the same
    arithmetic per point, so the layered propagation is bitwise the same (a remainder of the steps
    takes the 4/2/1-step passes), and both match the oracle."""
    import paratime_b200 as B

    hy, hx = 1 / ny, 1 / nx
    c, zy, zx, state = _case(ny, nx, hy, hx, w, batch, seed=ny + nx + steps)
    dt = 0.5 * min(hy, hx) / np.sqrt(2)
    prop = B.PmlPropagator(ctx, B.Grid((ny, nx), (hy, hx)), c, zy, zx, dt, steps)
    out = {}
    for sup in ("1", "0"):
        monkeypatch.setenv("PTB_PML_SUPER", sup)
        t = [ctx.tensor(a) for a in state]
        prop.propagate(*t)
        out[sup] = [x.cpu().numpy() for x in t]
    for a, b in zip(out["1"], out["0"]):
        assert np.array_equal(a, b)
    want = M.pml_steps(*(s_[:1] for s_ in state), M.PmlCoefficients(c, hy, hx, dt, zy, zx), steps)
    for got, ref in zip(out["1"], want):
        assert _rel(got[:1], ref) <= TOL


@pytest.mark.parametrize("n,w,steps", [(256, 32, 12), (512, 32, 10), (384, 16, 8)])
def test_interior_wavefront_equals_plain_tiles_bitwise(ctx, n, w, steps, monkeypatch):
    """The undamped interior runs the periodic wavefront kernel (k_wave2 on the interior
    rectangle) and the layer band-shaped tiles (frame mode), or k_wave2 on the plain-tile rectangle
    with 70 x 54 layer tiles, or k_pml_plain + layer tiles: the same arithmetic per point, so the
    layered propagation is bitwise the same in all three (steps not a multiple of 4 take a 2- or
    1-step pass)."""
    import paratime_b200 as B

    c, zy, zx, state = _case(n, n, 1 / n, 1 / n, w, 2, seed=n + w)
    prop = B.PmlPropagator(ctx, B.Grid((n, n), (1 / n, 1 / n)), c, zy, zx, 0.5 / n / np.sqrt(2), steps)
    out = {}
    for mode, wave, frame in (("frame", "1", "1"), ("tiles+wave", "1", "0"), ("tiles", "0", "0")):
        monkeypatch.setenv("PTB_PML_WAVE", wave)
        monkeypatch.setenv("PTB_PML_FRAME", frame)
        t = [ctx.tensor(a) for a in state]
        prop.propagate(*t)
        out[mode] = [x.cpu().numpy() for x in t]
    for other in ("tiles+wave", "tiles"):
        for a, b in zip(out["frame"], out[other]):
            assert np.array_equal(a, b), other
    out["1"] = out["frame"]
    want = M.pml_steps(*(s_[0] for s_ in state), M.PmlCoefficients(c, 1 / n, 1 / n, 0.5 / n / np.sqrt(2), zy, zx), steps)
    for got, ref in zip(out["1"], want):
        assert _rel(got[0], ref) <= TOL
