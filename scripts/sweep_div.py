import math, os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paratime_b200 as B
from workloads import cfg5_medium, cfg5_pulses
ctx = B.Context(0)
cases = [tuple(int(x) for x in a.split('x')) for a in sys.argv[1:]] or [(1024, 64), (256, 64), (512, 64)]
for n, batch in cases:
    c = cfg5_medium(n)
    dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
    prop = B.Propagator(ctx, B.Grid((n, n), (1.0 / n, 1.0 / n)), c, dt, 64)
    u = torch.as_tensor(cfg5_pulses(n, batch), device="cuda")
    v = torch.zeros_like(u)
    res = []
    for w in (0, 64, 96, 128, 192, 256):
        for div in (0, 1, 2, 3, 4, 6, 8, 16):
            os.environ["PTB_WAVE_W"] = str(w)
            os.environ["PTB_WAVE_DIV"] = str(div)
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
                res.append((round(batch * n * n * 64 / ms / 1e6), w, div, prop.plan(batch)))
            except Exception as ex:
                pass
    os.environ["PTB_WAVE_W"] = "0"; os.environ["PTB_WAVE_DIV"] = "0"
    res.sort(reverse=True)
    if os.environ.get("SWEEP_ALL"):
        for r in res:
            print("   ", r[0], r[1], r[2], r[3][:60], flush=True)
    print(n, batch, "auto:", [r for r in res if r[1] == 0 and r[2] == 0][:1], "best:", res[:4], flush=True)
