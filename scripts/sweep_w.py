"""Time k_wave2 strip widths per grid/batch (FAST, 64 steps): planner choice vs forced W."""
import math, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paratime_b200 as B
from workloads import cfg5_medium, cfg5_pulses
ctx = B.Context(0)
cases = [(128, 64), (128, 512), (256, 64), (512, 64), (512, 256), (1024, 64), (2048, 64), (4096, 16), (4096, 64)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
for n, batch in cases:
    c = cfg5_medium(n)
    dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
    prop = B.Propagator(ctx, B.Grid((n, n), (1.0 / n, 1.0 / n)), c, dt, 64)
    u = torch.as_tensor(cfg5_pulses(n, batch), device="cuda")
    v = torch.zeros_like(u)
    row = {}
    for w in (0, 64, 96, 128, 160, 192, 256):
        os.environ["PTB_WAVE_W"] = str(w)
        try:
            prop.propagate(u, v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                prop.propagate(u, v)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            row["auto" if w == 0 else w] = round(batch * n * n * 64 / ms / 1e6)  # Gupd/s
        except Exception as ex:
            row[w] = str(ex)[:40]
    os.environ["PTB_WAVE_W"] = "0"
    print(json.dumps({"grid": n, "batch": batch, "plan": prop.plan(batch), "Gupd_s": row}), flush=True)
    del u, v, prop
