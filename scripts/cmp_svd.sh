cd $GRAFT_REPO_ROOT
PYTHONPATH=. python tests/svd_probe.py 300 290 gpurun_out/coop.npz
PYTHONPATH=. PTB_JACOBI=single python tests/svd_probe.py 300 290 gpurun_out/single.npz
python - <<'P'
import numpy as np
for f in ["gpurun_out/coop.npz","gpurun_out/single.npz"]:
    a=np.load(f); m,U,S,V=a["m"],a["U"],a["S"],a["V"]
    ref=np.linalg.svd(m,compute_uv=False)
    print(f, "sv err", np.max(np.abs(S-ref)/ref[0]), "recon", np.linalg.norm(m-(U*S)@V.T)/np.linalg.norm(m), "orthV", np.max(np.abs(V.T@V-np.eye(V.shape[1]))), "orthU", np.max(np.abs(U.T@U-np.eye(U.shape[1]))))
a=np.load("gpurun_out/coop.npz"); b=np.load("gpurun_out/single.npz")
print("S diff", np.max(np.abs(a["S"]-b["S"])), "U diff", np.max(np.abs(np.abs(a["U"])-np.abs(b["U"]))))
P
