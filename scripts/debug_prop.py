import os, sys, math, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pass
import torch
import paratime_b200 as B
from oracle import paratime_np as P
ctx = B.Context(0)
def run(n, steps, mode, batch=1, seed=0):
    g = P.Grid(n, tuple(1.0/k for k in n))
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1,1,(batch,)+g.shape); v = rng.uniform(-1,1,(batch,)+g.shape)
    c = 0.5 + 0.5*rng.random(g.shape)
    dt = 0.9*min(g.h)/(math.sqrt(g.dim)*c.max())
    ref = P.verlet_steps(u, v, c, g, dt, steps)
    pr = B.Propagator(ctx, B.Grid(g.n, g.h), c, dt, steps)
    tu, tv = ctx.tensor(u), ctx.tensor(v)
    try:
        pr.propagate(tu, tv, mode=mode)
    except Exception as e:
        print(n, steps, mode, "ERROR", e); return
    gu = tu.cpu().numpy(); gv = tv.cpu().numpy()
    du = np.abs(gu-ref[0]); dv = np.abs(gv-ref[1])
    bad = np.argwhere(du > 0)
    print(n, steps, "exact" if mode else "fast", "maxdu %.3g maxdv %.3g nbad %d" % (du.max(), dv.max(), len(bad)), "first bad", bad[:5].tolist(), "unchanged", np.array_equal(gu, u))
for n, steps in [((64,64),1), ((64,64),2), ((4096,),1), ((48,64),1), ((128,128),1), ((128,128),8), ((200,96),1)]:
    run(n, steps, B.EXACT)
    run(n, steps, B.FAST)
