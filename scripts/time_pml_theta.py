"""Device theta-parareal with the absorbing layer on config 4 (workloads.cfg4_pml): iteration times.
python scripts/time_pml_theta.py [K [REPEATS]]   (PTB_PROF=1 prints the phase timeline to stderr)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paratime_b200 as B
from workloads import cfg4_pml

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = B.Context(0)
spec, c, cc, u0, v0, (zf, zc) = cfg4_pml()
nf, nc = spec["fine_n"][0], spec["coarse_n"][0]
gf = B.Grid((nf, nf), (1.0 / nf, 1.0 / nf))
gc = B.Grid((nc, nc), (1.0 / nc, 1.0 / nc))
fine = B.PmlPropagator(ctx, gf, c, zf, zf, spec["dt_fine"], spec["m_fine"])
coarse = B.PmlPropagator(ctx, gc, cc, zc, zc, spec["dt_coarse"], spec["m_coarse"])
tr = B.Transfer(ctx, gc, gf, spec["interp"])
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    r = B.pml_theta_run(fine, coarse, tr, spec["n_couplings"], K, u0, v0, tol=spec["tol"], scheme=spec["scheme"])
    print(json.dumps({"iteration_ms": [round(float(x), 2) for x in r["iteration_ms"]], "rank": [int(x) for x in r["rank"]]}), flush=True)
