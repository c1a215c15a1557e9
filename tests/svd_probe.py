"""Subprocess helper for tests/test_gpu_jacobi.py: thin SVD of a seeded p x q matrix through
ptb_thin_svd, saved to an .npz (the Jacobi path is chosen by PTB_JACOBI, read once per process)."""
import ctypes as C
import sys

import numpy as np
import torch

import paratime_b200 as B


def main(p, q, out):
    rng = np.random.default_rng(p * 1000 + q)
    k = min(p, q)
    u, _ = np.linalg.qr(rng.standard_normal((p, k)))
    v, _ = np.linalg.qr(rng.standard_normal((q, k)))
    s = np.logspace(0, -9, k)
    m = (u * s) @ v.T
    ctx = B.Context(0)
    M = torch.tensor(np.asfortranarray(m).ravel(order="F"), device="cuda")
    U = torch.empty(p * k, dtype=torch.float64, device="cuda")
    V = torch.empty(q * k, dtype=torch.float64, device="cuda")
    S = np.empty(k)
    lib = B.lib()
    B.api.check(lib.ptb_thin_svd(ctx.h, C.c_size_t(p), C.c_size_t(q), C.c_void_p(M.data_ptr()),
                                 C.c_void_p(U.data_ptr()), S.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.c_void_p(V.data_ptr())))
    np.savez(out, m=m, U=U.cpu().numpy().reshape(k, p).T, S=S, V=V.cpu().numpy().reshape(k, q).T)


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3])
