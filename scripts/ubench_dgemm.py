"""The hand-written DGEMM (ptb_dgemm, csrc/gemm.cu: DMMA tiles and DFMA register tiles) against cuBLAS's
DMMA kernels (torch float64 matmul, measurement only) on the corrector's shapes.

Shapes (column-major BLAS view, rows = 3 N_c of config 4 = 196608, r ~ 150, N = 128):
  TN  U^T F            m=r   n=N    k=rows   (split-K)
  NN  F - U (U^T F)    m=rows n=N   k=r
  NN  [U Q_F] Xh       m=rows n=r   k=r+N
  NT  H = L R^T        m=r+N n=r+N  k=N
  TN  S = V^T V        m=32  n=32   k=rows
Prints one JSON line per shape: ms and TFLOP/s for both."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paratime_b200 as B  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
ctx = B.Context(0)
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 196608
SHAPES = [("U^T F", 1, 0, 150, 128, rows), ("F - U(U^T F)", 0, 0, rows, 128, 150),
          ("[U Q_F] Xh", 0, 0, rows, 150, 278), ("H = L R^T", 0, 1, 278, 278, 128), ("V^T V", 1, 0, 32, 32, rows)]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, ta, tb, m, n, k in SHAPES:
    A = torch.randn((m, k) if ta else (k, m), dtype=torch.float64, device="cuda")  # row-major of the col-major
    Bm = torch.randn((k, n) if tb else (n, k), dtype=torch.float64, device="cuda")
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda")
    lda, ldb = (k if ta else m), (n if tb else k)
    dp = ctypes.c_void_p

    def ours():
        B.api.check(B.lib().ptb_dgemm(ctx.h, ta, tb, m, n, k, ctypes.c_double(1.0), dp(A.data_ptr()), lda,
                                      dp(Bm.data_ptr()), ldb, ctypes.c_double(0.0), dp(C.data_ptr()), m))

    # a column-major X (r x c) is the row-major torch tensor (c x r): X = tensor^T
    Acm = A.t()
    opA = Acm.t() if ta else Acm
    Bcm = Bm.t()
    opB = Bcm.t() if tb else Bcm

    def cublas():
        torch.matmul(opA, opB)

    reps = 5 if m * n * k > 1e9 else 50
    os.environ["PTB_DGEMM"] = "dmma"
    t_o = timed(ours, reps)
    os.environ["PTB_DGEMM"] = "dfma"
    t_f = timed(ours, reps)
    os.environ.pop("PTB_DGEMM")
    t_c = timed(cublas, reps)
    fl = 2.0 * m * n * k
    print(json.dumps({"shape": name, "m": m, "n": n, "k": k, "ours_dmma_ms": round(t_o, 4),
                      "ours_dmma_tflops": round(fl / t_o / 1e9, 2), "ours_dfma_ms": round(t_f, 4),
                      "ours_dfma_tflops": round(fl / t_f / 1e9, 2), "cublas_dmma_ms": round(t_c, 4),
                      "cublas_tflops": round(fl / t_c / 1e9, 2)}), flush=True)
