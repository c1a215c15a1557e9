# round-2 session-5 call C: launch list of one layered coupling (2048^2 x 16 slices, 32-cell layer)
cat > /tmp/pml_one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paratime_b200 as B
ctx = B.Context(0)
n, w, batch, steps = 2048, 32, 16, 16
h = 1 / n
zs = B.damping_profile(n, w, h, 1.0, 1e-4)
g = B.Grid((n, n), (h, h))
pml = B.PmlPropagator(ctx, g, np.ones((n, n)), zs, zs, h / 8, steps)
t = [torch.zeros((batch, n, n), dtype=torch.float64, device="cuda:0") for _ in range(4)]
t[0].normal_()
for _ in range(3):
    pml.propagate(*t)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv --log-file gpurun_out/r02cc_pml_launches.csv python /tmp/pml_one.py > gpurun_out/r02cc_ncu.log 2>&1
tail -3 gpurun_out/r02cc_ncu.log
