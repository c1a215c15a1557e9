"""World-size-2 gloo test (CPU) of the slice-sharded decomposition of the absorbing-layer plain
parareal (csrc/pml.cu pml_parareal with a communicator): all-gather of the coarse payload,
replicated sweep, own combine and boundary send must reproduce the one-process oracle
(oracle/pml_np.plain_parareal) bitwise."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    from tests.test_pml_oracle import _small_parareal

    s = _small_parareal(0, N=5, K=3)
    return s


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.sharded_oracle import pml_plain_sharded

    s = _setup()
    hist = pml_plain_sharded(s["u0"], np.zeros_like(s["u0"]), s["kf"], s["mf"], s["kc"], s["mc"], s["t"], s["N"],
                             s["K"])
    q.put((rank, [{n: np.stack(st) for n, st in h.items()} for h in hist]))
    dist.destroy_process_group()


def test_pml_sharded_decomposition_matches_oracle():
    from oracle import pml_np as M

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, hist = q.get(timeout=300)
        got[r] = hist
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = _setup()
    its, _ = M.plain_parareal(s["u0"], np.zeros_like(s["u0"]), s["kf"], s["mf"], s["kc"], s["mc"], s["t"], s["N"],
                              s["K"])
    for k in range(s["K"]):
        for r in range(world):
            for n, st in got[r][k].items():
                assert np.array_equal(st, np.stack(its[k][n])), (k, r, n)
