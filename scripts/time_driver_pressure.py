"""Warm driver timings (second run on one context) after torch has reserved and cached large
device buffers, as in bench.py:  python scripts/time_driver_pressure.py GIB cfg...  """
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paratime_b200 as B
import workloads as W
x = torch.empty(int(sys.argv[1]) * (1 << 27), dtype=torch.float64, device="cuda")  # GiB
x.fill_(1.0)
del x
ctx = B.Context(0)
for cfg in [int(a) for a in sys.argv[2:]] or [1, 2]:
    spec, cf, cc, u0, v0 = W.CONFIGS[cfg]()
    B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0)
    r = B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0)
    t = r["times"]
    med = lambda k: round(sorted(t[k])[len(t[k]) // 2], 2)
    print(cfg, {k: med(k) for k in ("iteration_ms", "parallel_ms", "procrustes_ms", "sweep_ms", "finalize_ms")},
          [round(v, 2) for v in t["iteration_ms"]])
