"""Time the device theta-parareal on BASELINE configs 1-4 (args "cfg[:K]") (and optionally compare with the oracle/_ref)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paratime_b200 as B
import workloads as W
ctx = B.Context(0)
for arg in (sys.argv[1:] or ["1", "2", "3"]):
    cfg, _, kk = arg.partition(":")  # "cfg[:K]"
    cfg = int(cfg)
    spec, cf, cc, u0, v0 = W.CONFIGS[cfg]()
    if kk:
        spec["iterations"] = int(kk)
    t0 = time.time()
    r = B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0)
    wall = time.time() - t0
    t = r["times"]
    print(json.dumps({"cfg": cfg, "wall_s": round(wall, 3), "reference_ms": round(t["reference_ms"], 2),
                      "iteration_ms": [round(x, 2) for x in t["iteration_ms"]],
                      "parallel_ms": [round(x, 2) for x in t["parallel_ms"]], "gather_ms": [round(x, 3) for x in t["gather_ms"]],
                      "procrustes_ms": [round(x, 2) for x in t["procrustes_ms"]],
                      "sweep_ms": [round(x, 2) for x in t["sweep_ms"]],
                      "finalize_ms": [round(x, 2) for x in t["finalize_ms"]],
                      "rank": r["rank"].tolist(), "final_err": r["energy_err"][:, -1].round(6).tolist()}), flush=True)
