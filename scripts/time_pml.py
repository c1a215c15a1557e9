"""Device timing of the absorbing-layer propagator vs the periodic FAST kernel (CUDA events)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paratime_b200 as B

ctx = B.Context(0)
out = []
for n, w, batch, steps in [(2048, 32, 16, 128), (2048, 32, 64, 64), (256, 4, 128, 8), (512, 32, 64, 64)]:
    h = 1 / n
    c = np.ones((n, n))
    zs = B.damping_profile(n, w, h, 1.0, 1e-4)
    g = B.Grid((n, n), (h, h))
    pml = B.PmlPropagator(ctx, g, c, zs, zs, h / 8, steps)
    per = B.Propagator(ctx, g, c, h / 8, steps)
    t = [torch.zeros((batch, n, n), dtype=torch.float64, device="cuda:0") for _ in range(4)]
    t[0].normal_()
    rec = {"grid": n, "layer": w, "batch": batch, "steps": steps}
    for name, fn in [("pml", lambda: pml.propagate(*t)), ("periodic", lambda: per.propagate(t[0], t[1], mode=B.FAST))]:
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        rec[name + "_ms"] = ms
        rec[name + "_upd_s"] = batch * n * n * steps / (ms * 1e-3)
    out.append(rec)
    print(json.dumps(rec), flush=True)
