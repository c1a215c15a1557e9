"""Warm timings of the Procrustes building blocks through the C ABI (ptb_truncated_qr,
ptb_thin_svd) on the shapes the parareal configs produce: CUDA events around N repeated calls
after warm-up (each call includes its host sync, as in update_svd).

  python scripts/ubench_procrustes.py            # all shapes
  PTB_QR=blocked python scripts/ubench_procrustes.py qr
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paratime_b200 as B

QR_SHAPES = [(3072, 16), (12288, 32), (49152, 64), (196608, 128)]
SVD_SHAPES = [(32, 32), (60, 60), (80, 80), (95, 95), (108, 108), (160, 160)]


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(which):
    ctx = B.Context(0)
    lib = B.lib()
    rng = np.random.default_rng(1)
    out = {}
    if which in ("all", "qr"):
        for m, n in QR_SHAPES:
            a = rng.standard_normal((m, n)) * np.logspace(0, -8, n)[None, :]
            A = torch.tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
            Q = torch.zeros(m * n, dtype=torch.float64, device="cuda")
            R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
            keep = C.c_size_t()
            tol = 1e-14 * float(np.linalg.norm(a))

            def call():
                B.api.check(lib.ptb_truncated_qr(ctx.h, C.c_size_t(m), C.c_size_t(n), C.c_void_p(A.data_ptr()),
                                                 C.c_double(tol), C.c_void_p(Q.data_ptr()), C.c_void_p(R.data_ptr()),
                                                 C.byref(keep)))

            out[f"qr {m}x{n}"] = round(timed(call), 4)
    if which in ("all", "svd"):
        for p, q in SVD_SHAPES:
            k = min(p, q)
            u, _ = np.linalg.qr(rng.standard_normal((p, k)))
            v, _ = np.linalg.qr(rng.standard_normal((q, k)))
            mm = (u * np.logspace(0, -12, k)) @ v.T
            M = torch.tensor(np.asfortranarray(mm).ravel(order="F"), device="cuda")
            U = torch.empty(p * k, dtype=torch.float64, device="cuda")
            V = torch.empty(q * k, dtype=torch.float64, device="cuda")
            S = np.empty(k)

            def call():
                B.api.check(lib.ptb_thin_svd(ctx.h, C.c_size_t(p), C.c_size_t(q), C.c_void_p(M.data_ptr()),
                                             C.c_void_p(U.data_ptr()), S.ctypes.data_as(C.POINTER(C.c_double)),
                                             C.c_void_p(V.data_ptr())))

            out[f"svd {p}x{q}"] = round(timed(call, reps=10), 4)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PTB_")}, "ms": out}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
