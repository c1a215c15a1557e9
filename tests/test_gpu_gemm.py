"""The hand-written DGEMM / DGEMV (csrc/gemm.cu, DMMA and DFMA families) against numpy on the corrector's shapes.

Every Eigen product of the reference's Procrustes step (procrustes.cpp:65-66, 201-234, 251) and
PhaseCorrector::apply (:82-86) runs through it: tall-skinny transposed products with split-K
(k = 3 N_c up to 196608), tall rotations, small dense products, matrix-vector products; all four
transpose cases, leading dimensions larger than the rows, beta = 0 / 1 / other."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # (ta, tb, m, n, k)
    (1, 0, 46, 64, 49152),     # U^T F at config 3 (split-K)
    (1, 0, 150, 128, 196608),  # U^T F at config 4 scale (split-K)
    (0, 0, 49152, 46, 90),     # [U Q_F] Xh rotation
    (0, 0, 3000, 70, 33),
    (0, 1, 90, 80, 64),        # H = L R^T
    (1, 1, 37, 29, 71),
    (0, 1, 513, 65, 17),
    (0, 0, 65536, 1, 150),     # Z dz (GEMV)
    (1, 0, 150, 1, 196608),    # Y^T v (GEMV^T)
    (1, 0, 1, 1, 5),
    (0, 1, 150, 100, 64),      # short m: DMMA computes C^T with a transposed store
    (0, 0, 200, 60, 300),
    (1, 1, 150, 90, 77),
    (0, 0, 7, 3, 0),           # k = 0: C = beta C
]


def _run(ta, tb, m, n, k, alpha, beta, pad, seed):
    import torch

    import paratime_b200 as B

    ctx = B.Context(0)
    rng = np.random.default_rng(seed)
    ar, ac = (k, m) if ta else (m, k)
    br, bc = (n, k) if tb else (k, n)
    lda, ldb, ldc = ar + pad, br + pad, m + pad
    A = rng.standard_normal((ac, lda))  # column-major storage: rows are columns
    Bm = rng.standard_normal((bc, ldb))
    C = rng.standard_normal((n, ldc))
    opA = (A[:, :ar].T)
    opA = opA.T if ta else opA
    opB = Bm[:, :br].T
    opB = opB.T if tb else opB
    want = alpha * (opA @ opB) + (beta * C[:, :m].T if beta != 0 else 0.0)
    tA, tB, tC = (torch.as_tensor(x, device="cuda") for x in (A, Bm, C))
    dp = ctypes.c_void_p
    B.api.check(B.lib().ptb_dgemm(ctx.h, ta, tb, m, n, k, ctypes.c_double(alpha), dp(tA.data_ptr()), lda,
                                  dp(tB.data_ptr()), ldb, ctypes.c_double(beta), dp(tC.data_ptr()), ldc))
    got = tC.cpu().numpy()
    assert np.array_equal(got[:, m:], C[:, m:]), "wrote outside the m rows"
    return got[:, :m].T, want, k


@pytest.mark.parametrize("family", ["dmma", "dfma"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (-1.0, 1.0), (0.5, -2.0)])
def test_dgemm_matches_numpy(shape, alpha, beta, family, monkeypatch):
    """Both kernel families: k_dgemm_mma (fp64 tensor cores, the default) and k_dgemm (DFMA)."""
    monkeypatch.setenv("PTB_DGEMM", family)
    got, want, k = _run(*shape, alpha, beta, pad=3, seed=sum(shape))
    scale = np.sqrt(max(k, 1)) * (abs(alpha) + abs(beta)) * 4
    assert np.max(np.abs(got - want)) <= 1e-15 * scale * max(1.0, np.max(np.abs(want))) + 1e-300


def test_dgemm_beta_zero_ignores_nan_in_c():
    import torch

    import paratime_b200 as B

    ctx = B.Context(0)
    A = torch.ones((4, 8), dtype=torch.float64, device="cuda")
    Bm = torch.ones((3, 4), dtype=torch.float64, device="cuda")
    C = torch.full((3, 8), float("nan"), dtype=torch.float64, device="cuda")
    dp = ctypes.c_void_p
    B.api.check(B.lib().ptb_dgemm(ctx.h, 0, 0, 8, 3, 4, ctypes.c_double(1.0), dp(A.data_ptr()), 8,
                                  dp(Bm.data_ptr()), 4, ctypes.c_double(0.0), dp(C.data_ptr()), 8))
    assert torch.all(C == 4.0)


def test_dgemm_split_k_is_deterministic():
    a = _run(1, 0, 64, 64, 196608, 1.0, 0.0, pad=0, seed=3)[0]
    b = _run(1, 0, 64, 64, 196608, 1.0, 0.0, pad=0, seed=3)[0]
    assert np.array_equal(a, b)
