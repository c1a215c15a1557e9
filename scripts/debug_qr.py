import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, scipy.linalg
import paratime_b200 as B
from paratime_b200.api import _ptr, check, lib
ctx = B.Context(0)
rng = np.random.default_rng(0)
for (m, n) in [(24, 4), (768, 16), (3072, 16), (2000, 33), (700, 40)]:
    A = rng.standard_normal((m, n))
    A[:, 3] = A[:, 1]  # rank deficiency
    t = torch.as_tensor(A.T.copy(), device="cuda")
    Q = torch.zeros(m * n, dtype=torch.float64, device="cuda"); R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    keep = C.c_size_t()
    check(lib().ptb_truncated_qr(ctx.h, C.c_size_t(m), C.c_size_t(n), _ptr(t), C.c_double(1e-10), _ptr(Q), _ptr(R), C.byref(keep)))
    k = keep.value
    Qh = Q.cpu().numpy()[: m * k].reshape(k, m).T; Rh = R.cpu().numpy()[: k * n].reshape(n, k).T
    Qo, Ro, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
    print(m, n, "keep", k, "| QR - A|", np.max(np.abs(Qh @ Rh - A)), "orth", np.max(np.abs(Qh.T @ Qh - np.eye(k))),
          "diag", np.abs(np.diag(Rh[:, :])).round(3)[:4] if False else "")
for (p, q) in [(16, 16), (5, 7), (40, 33), (100, 100), (64, 80)]:
    M = rng.standard_normal((p, q))
    t = torch.as_tensor(M.T.copy(), device="cuda")
    k = min(p, q)
    U = torch.zeros(p * k, dtype=torch.float64, device="cuda"); V = torch.zeros(q * k, dtype=torch.float64, device="cuda")
    S = np.zeros(k)
    check(lib().ptb_thin_svd(ctx.h, C.c_size_t(p), C.c_size_t(q), _ptr(t), _ptr(U), S.ctypes.data_as(C.POINTER(C.c_double)), _ptr(V)))
    Uh = U.cpu().numpy().reshape(k, p).T; Vh = V.cpu().numpy().reshape(k, q).T
    so = np.linalg.svd(M, compute_uv=False)
    print("svd", p, q, "sigma err", np.max(np.abs(S - so)), "recon", np.max(np.abs(Uh @ np.diag(S) @ Vh.T - M)), "orthU", np.max(np.abs(Uh.T@Uh - np.eye(k))))
