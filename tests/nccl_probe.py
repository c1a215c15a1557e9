"""Subprocess helper for tests/test_gpu_sharded.py: cfg1 theta-parareal through a one-rank NCCL
communicator (PTB_NCCL_FORCE=1 makes world 1 create a real ncclComm_t)."""
import sys

import numpy as np

import paratime_b200 as B
import workloads as W

spec, cf, cc, u0, v0 = W.cfg1()
ctx = B.Context(0)
comm = B.api.Comm(ctx, 0, 1)
r = B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, keep_states=True, comm=comm)
np.savez(sys.argv[1], states=r["states"], energy_err=r["energy_err"], rank=r["rank"])
