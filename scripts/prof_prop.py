"""Minimal K1 driver for ncu: python scripts/prof_prop.py GRID BATCH REPS [fast|exact]"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paratime_b200 as B
from workloads import cfg5_medium, cfg5_pulses
n = int(sys.argv[1]); batch = int(sys.argv[2]); reps = int(sys.argv[3]); mode = B.EXACT if len(sys.argv) > 4 and sys.argv[4] == "exact" else B.FAST
ctx = B.Context(0)
c = cfg5_medium(n)
dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
prop = B.Propagator(ctx, B.Grid((n, n), (1.0 / n, 1.0 / n)), c, dt, 64)
u = torch.as_tensor(cfg5_pulses(n, batch), device="cuda"); v = torch.zeros_like(u)
for _ in range(reps):
    prop.propagate(u, v, mode=mode)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); prop.propagate(u, v, mode=mode); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"grid {n} batch {batch}: {ms:.3f} ms  {batch*n*n*64/ms/1e9:.1f} Gupd/s  launches {ctx.launches()}")
