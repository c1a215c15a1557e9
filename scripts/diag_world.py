import sys, threading, traceback, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paratime_b200 as B
import workloads as W
world = int(sys.argv[1])
spec, cf, cc, u0, v0 = W.cfg2(); spec = dict(spec, iterations=3)
group = B.api.LoopbackGroup(world)
ctxs = [B.Context(0) for _ in range(world)]
comms = [group.comm(ctxs[r], r) for r in range(world)]
def work(r):
    try:
        B.api.parareal_run(ctxs[r], B.api.run_spec(**spec), cf, cc, u0, v0, keep_states=True, comm=comms[r])
        print("rank", r, "done", flush=True)
    except Exception as e:
        print("rank", r, "ERROR", e, flush=True); os._exit(3)
ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
