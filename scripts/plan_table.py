"""Print the propagate() launch plan for the BASELINE workloads (no GPU work beyond planning)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paratime_b200 as B
ctx = B.Context(0)
for n, batch, steps in [(128, 64, 64), (256, 64, 64), (512, 64, 64), (512, 64, 8), (1024, 64, 64), (2048, 1, 128),
                        (2048, 16, 64), (2048, 64, 64), (2048, 128, 128), (4096, 16, 64), (4096, 64, 64)]:
    c = np.ones((n, n))
    p = B.Propagator(ctx, B.Grid((n, n), (1 / n, 1 / n)), c, 0.1 / n, steps)
    print(n, batch, steps, p.plan(batch, B.FAST))
