"""The slice-sharded driver (the multi-GPU path) against the one-GPU run.

Ranks are in-process threads with their own contexts on cuda:0 joined by the loopback
communicator (host rendezvous + cudaMemcpy), so the C++ sharding logic — partition,
coarse-payload all-gather, replicated Procrustes + sweep, per-rank fine combine, boundary
exchange — runs unchanged with world = 2, 3, 4 on one GPU without device-side waits.
Every replicated step is deterministic, so results must be bitwise identical to world = 1."""
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _run_world(world, spec, cf, cc, u0, v0):
    import paratime_b200 as B

    group = B.api.LoopbackGroup(world)
    ctxs = [B.Context(0).use_own_stream() for _ in range(world)]  # a stream per rank
    comms = [group.comm(ctxs[r], r) for r in range(world)]
    out = [None] * world
    err = []

    def work(r):
        try:
            out[r] = B.api.parareal_run(ctxs[r], B.api.run_spec(**spec), cf, cc, u0, v0, keep_states=True,
                                        comm=comms[r])
        except Exception as e:  # pragma: no cover
            err.append(e)

    # daemon threads joined with a timeout: a rank that fails leaves the others waiting at the
    # loopback barrier, and the failure must surface instead of hanging the suite
    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not err, err
    assert all(not t.is_alive() for t in ts), "a rank did not finish (loopback barrier)"
    return out


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("variant,large", [(1, False), (0, False), (1, True)])
def test_sharded_equals_single_gpu(world, variant, large, monkeypatch):
    """large: the sweep's large-corrector branch (config 4's), whose GEMVs are row-sharded over
    the ranks (fixed row blocks, fixed-order sums): still bitwise the one-GPU result."""
    if large:
        monkeypatch.setenv("PTB_FUSED_SWEEP_MAX", "0")
    spec, cf, cc, u0, v0 = W.cfg1(tol=1e-8)
    spec = dict(spec, variant=variant, iterations=3)
    single = _run_world(1, spec, cf, cc, u0, v0)[0]
    outs = _run_world(world, spec, cf, cc, u0, v0)
    N = spec["n_couplings"]
    chunk = -(-N // world)
    for r, o in enumerate(outs):
        assert np.array_equal(o["energy_err"], single["energy_err"])
        assert np.array_equal(o["l2_err"], single["l2_err"])
        assert list(o["rank"]) == list(single["rank"])
        np.testing.assert_array_equal(o["residual"][1:], single["residual"][1:])
        a = 1 + r * chunk
        b = min(N + 1, a + chunk)
        lo = 0 if r == 0 else a
        assert np.array_equal(o["states"][:, lo:b], single["states"][:, lo:b])


@pytest.mark.parametrize("world", [2, 3, 4])
def test_row_sharded_procrustes_equals_single_gpu(world):
    """Config 2 (3 N_c = 12288 rows = 48 slabs of one TSQR leaf): update_svd runs row-sharded —
    the U^T F / V^T G partials per fixed slab gathered and summed in slab order, each rank's TSQR
    leaves factored by it and the leaves' R stack gathered, the new factors' own rows gathered.
    Iterates, error tables, ranks and residuals bitwise equal to one GPU; the one-GPU run takes the
    same slab path (tests/test_gpu_configs.py pins it to the reference at 1e-10)."""
    spec, cf, cc, u0, v0 = W.cfg2()
    spec = dict(spec, iterations=3)
    single = _run_world(1, spec, cf, cc, u0, v0)[0]
    outs = _run_world(world, spec, cf, cc, u0, v0)
    N = spec["n_couplings"]
    chunk = -(-N // world)
    for r, o in enumerate(outs):
        assert list(o["rank"]) == list(single["rank"])
        assert np.array_equal(o["energy_err"], single["energy_err"])
        np.testing.assert_array_equal(o["residual"][1:], single["residual"][1:])
        a = 1 + r * chunk
        b = min(N + 1, a + chunk)
        lo = 0 if r == 0 else a
        assert np.array_equal(o["states"][:, lo:b], single["states"][:, lo:b])


@pytest.mark.timeout(420)
def test_nccl_communicator_world1_equals_no_comm(tmp_path):
    """The NCCL runtime path (dlopen of libnccl.so.2, ncclCommInitRank, ncclAllGather of the
    coarse payload) on one GPU: a one-rank NCCL communicator must give bitwise the result of
    the communicator-free run.  Multi-rank NCCL needs several GPUs (bench.py under torchrun)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    import paratime_b200 as B

    root = Path(__file__).resolve().parent.parent
    out = tmp_path / "nccl.npz"
    # one process, one GPU: keep NCCL's bootstrap on loopback (a box without a routable interface
    # once stalled the probe's ncclCommInitRank past the suite's budget)
    env = dict(os.environ, PTB_NCCL_FORCE="1", PYTHONPATH=str(root), NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")
    subprocess.run([sys.executable, str(root / "tests" / "nccl_probe.py"), str(out)], check=True, env=env,
                   timeout=360)
    got = np.load(out)
    spec, cf, cc, u0, v0 = W.cfg1()
    ctx = B.Context(0)
    ref = B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, keep_states=True)
    assert np.array_equal(got["states"], ref["states"])
    assert np.array_equal(got["energy_err"], ref["energy_err"])
    assert np.array_equal(got["rank"], ref["rank"])
