import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, scipy.linalg
import paratime_b200 as B
from paratime_b200.api import _ptr, check, lib
ctx = B.Context(0)
rng = np.random.default_rng(0)
for (m, n) in [(600, 6), (1100, 5)]:
    A = rng.standard_normal((m, n))
    t = torch.as_tensor(A.T.copy(), device="cuda")
    Q = torch.zeros(m * n, dtype=torch.float64, device="cuda"); R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    keep = C.c_size_t()
    check(lib().ptb_truncated_qr(ctx.h, C.c_size_t(m), C.c_size_t(n), _ptr(t), C.c_double(1e-10), _ptr(Q), _ptr(R), C.byref(keep)))
    k = keep.value
    Qh = Q.cpu().numpy()[: m * k].reshape(k, m).T; Rh = R.cpu().numpy()[: k * n].reshape(n, k).T
    Qo, Ro, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
    Runp = np.zeros_like(Ro); Runp[:, piv] = Ro
    print(m, n, "pivots scipy", piv, "diag scipy", np.abs(np.diag(Ro)).round(4))
    print("  gpu R\n", np.abs(Rh).round(4))
    print("  ref R\n", np.abs(Runp).round(4))
    print("  |QtA - R|", np.max(np.abs(Qh.T @ A - Rh)), " Q vs Qo (abs)", np.max(np.abs(np.abs(Qh.T @ Qo) - np.eye(k))))
