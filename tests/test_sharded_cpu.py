"""World-size-2 gloo test (CPU) of the sharded parareal decomposition used by the
multi-GPU driver: coarse-only replicated sweep + per-rank fine combine + boundary exchange
must reproduce the reference's theta_engine (numpy oracle) iterates."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _small_setup():
    from oracle import paratime_np as P

    nf, nc, N = 32, 16, 6
    fg = P.Grid((nf, nf), (1 / nf, 1 / nf))
    cg = P.Grid((nc, nc), (1 / nc, 1 / nc))
    y, x = np.meshgrid(np.arange(nf) / nf, np.arange(nf) / nf, indexing="ij")
    c = 1.0 - 0.25 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)
    u0 = np.exp(-60 * ((x - 0.45) ** 2 + (y - 0.55) ** 2))
    dt_com = 1.0 / N / 4
    sch = P.Schedule(N * dt_com, dt_com, N, fg, c, dt_com / 16, 16, cg, c[::2, ::2].copy(), dt_com / 4, 4)
    t = P.Transfer(cg, fg, P.FOURIER)
    return (u0, np.zeros_like(u0)), sch, t


def _worker(rank, world, port, K, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.sharded_oracle import theta_sharded

    init, sch, t = _small_setup()
    hist = theta_sharded(init, sch, t, K, 0, 1e-8)
    q.put((rank, [{n: (s[0].tolist(), s[1].tolist()) for n, s in h.items()} for h in hist]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_decomposition_matches_reference_theta(world):
    from oracle import paratime_np as P

    K = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, hist = q.get(timeout=300)
        got[r] = hist
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    init, sch, t = _small_setup()
    ref = P.theta_parareal(init, sch, t, K, scheme=0, tol=1e-8)
    for k in range(K):
        for r in range(world):
            for n, (u, v) in got[r][k].items():
                ru, rv = ref.iterations[k + 1].states[int(n)]
                e = P.energy_error((np.array(u), np.array(v)), (ru, rv), sch.c_fine, sch.fine_grid, 0)
                assert e <= 1e-12, (k, n, e)


def _snapshots(seed, rows, cols, rank_true):
    """Snapshot pairs G, F = Q G + noise with a decaying spectrum (the corrector's regime)."""
    rng = np.random.default_rng(seed)
    basis = np.linalg.qr(rng.standard_normal((rows, rank_true)))[0]
    w = basis * (10.0 ** -np.linspace(0, 6, rank_true))
    G = w @ rng.standard_normal((rank_true, cols))
    rot = np.linalg.qr(rng.standard_normal((rank_true, rank_true)))[0]
    F = (basis @ rot * (10.0 ** -np.linspace(0, 6, rank_true))) @ rng.standard_normal((rank_true, cols))
    return F, G


def _rows_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import paratime_np as P
    from tests.sharded_oracle import update_svd_row_sharded

    rows, cols, leaf = 768, 12, 48
    corr = P.empty_corrector()
    out = []
    for it in range(3):
        F, G = _snapshots(100 + it, rows, cols, 20)
        corr = P.solve_from_scratch(F, G, 1e-8) if corr.empty() else update_svd_row_sharded(corr, F, G, 1e-8, leaf)
        out.append((corr.X.copy(), corr.S.copy(), corr.Y.copy()))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_update_svd_matches_reference(world):
    """The row-sharded update_svd decomposition (slab partial sums in slab order, per-rank TSQR
    leaves + gathered R stack, row-local projections/rotations) reproduces procrustes.cpp:188-237
    (oracle update_svd): same ranks, same singular values, same operator; ranks agree bitwise."""
    from oracle import paratime_np as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    corr = P.empty_corrector()
    for it in range(3):
        F, G = _snapshots(100 + it, 768, 12, 20)
        corr = P.update_svd(corr, F, G, 1e-8)
        X0, S0, Y0 = got[0][it]
        for r in range(1, world):  # replicated results are identical on every rank
            for a, b in zip(got[0][it], got[r][it]):
                assert np.array_equal(a, b)
        assert S0.size == corr.rank
        assert np.allclose(S0, corr.S, rtol=1e-10, atol=0)
        want = (corr.X * corr.S) @ corr.Y.T
        have = (X0 * S0) @ Y0.T
        assert np.linalg.norm(have - want) <= 1e-10 * np.linalg.norm(want)
        assert np.linalg.norm(X0.T @ X0 - np.eye(S0.size)) <= 1e-10
