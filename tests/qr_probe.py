"""Subprocess helper for tests/test_gpu_qr.py: ptb_truncated_qr on seeded tall matrices (the
QR path is chosen by PTB_QR, read once per process)."""
import ctypes as C
import sys

import numpy as np
import torch

import paratime_b200 as B


def mats():
    rng = np.random.default_rng(77)
    out = []
    for m, n, rank in [(4096, 40, 40), (6000, 64, 50), (20000, 100, 100), (3000, 33, 20), (8192, 96, 96),
                       (12288, 32, 29), (49152, 64, 60), (1537, 17, 17),
                       (30000, 128, 90), (16384, 72, 72), (20000, 100, 50)]:  # two-panel route, rank-deficient panels
        a = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
        a *= np.logspace(0, -6, n)[None, :]  # graded columns: pivoting matters
        out.append(a)
    # exactly repeated and zero columns, and columns supported on a few rows (zero reflectors
    # inside TSQR leaves)
    a = rng.standard_normal((20000, 48))
    a[:, 5] = a[:, 2]
    a[:, 11] = 0.0
    a[:, 20] = 0.0
    a[:300, 20] = rng.standard_normal(300)
    a[:, 30] = 2.0 * a[:, 7]
    out.append(a)
    # snapshot-like: whole TSQR leaves of tiny entries (rows far from the wave: squares underflow,
    # some entries denormal) stacked with O(1) rows -- the reflectors of those leaves must stay
    # orthogonal (config 3's first snapshot block exposed this)
    a = rng.standard_normal((49152, 64)) @ np.diag(np.logspace(0, -5, 64))
    a[3000:9000] *= 1e-160
    a[20000:26000] *= 1e-300
    a[40000:41000] *= 1e-310
    out.append(a)
    return out


def main(path):
    ctx = B.Context(0)
    lib = B.lib()
    res = {}
    for t, a in enumerate(mats()):
        m, n = a.shape
        A = torch.tensor(np.asfortranarray(a).ravel(order="F"), device="cuda")
        Q = torch.zeros(m * n, dtype=torch.float64, device="cuda")
        R = torch.zeros(n * n, dtype=torch.float64, device="cuda")
        keep = C.c_size_t()
        tol = 1e-14 * np.linalg.norm(a)
        B.api.check(lib.ptb_truncated_qr(ctx.h, C.c_size_t(m), C.c_size_t(n), C.c_void_p(A.data_ptr()), C.c_double(tol),
                                         C.c_void_p(Q.data_ptr()), C.c_void_p(R.data_ptr()), C.byref(keep)))
        k = keep.value
        res[f"A{t}"] = a
        res[f"Q{t}"] = Q.cpu().numpy()[: m * k].reshape(k, m).T
        res[f"R{t}"] = R.cpu().numpy()[: k * n].reshape(n, k).T
        res[f"tol{t}"] = tol
    np.savez(path, **res)


if __name__ == "__main__":
    main(sys.argv[1])
