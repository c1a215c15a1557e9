"""truncated_qr (procrustes.cpp:34-46) on tall snapshot-like blocks: the TSQR route (leaf QRs in
shared memory, then the pivoted QR of the last stack; n <= 64), the two-panel route (two TSQR
panels with block Gram-Schmidt between them, then the pivoted QR of the assembled R; 64 < n <=
128, the default there), the blocked route (unpivoted panel QR + WY updates, then the pivoted QR
of R1), the direct column-pivoted kernel and
the default choice must all reproduce the oracle's keep count, an orthonormal
Q and the same product Q R as the oracle's column-pivoted QR."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import paratime_np as P

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("path", ["auto", "blocked", "direct", "tsqr", "panel2"])
def test_truncated_qr_tall_matches_oracle(tmp_path, path):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    env.pop("PTB_QR", None)
    if path != "auto":
        env["PTB_QR"] = path
    out = tmp_path / "qr.npz"
    subprocess.run([sys.executable, str(ROOT / "tests" / "qr_probe.py"), str(out)], check=True, env=env, timeout=600)
    d = np.load(out)
    t = 0
    while f"A{t}" in d:
        a, q, r, tol = d[f"A{t}"], d[f"Q{t}"], d[f"R{t}"], float(d[f"tol{t}"])
        qo, ro = P.truncated_qr(a, tol)
        assert q.shape[1] == qo.shape[1], (t, q.shape, qo.shape)  # same keep decision
        k = q.shape[1]
        assert np.max(np.abs(q.T @ q - np.eye(k))) <= 1e-12
        scale = np.linalg.norm(a)
        assert np.linalg.norm(q @ r - qo @ ro) <= 1e-12 * scale, t
        if k == a.shape[1]:
            assert np.linalg.norm(q @ r - a) <= 1e-12 * scale, t
        t += 1


@pytest.mark.gpu
def test_two_panel_pair_equals_sequential_bitwise(monkeypatch):
    """update_svd on the row-slab path with 64 < columns <= 128 (config 4's N = 128 snapshots): F and
    G go through the two-panel TSQR route as a pair (shared leaf / stack / down-sweep launches) or
    one after the other (PTB_QR2_PAIR=0) — the same arithmetic per matrix, so the factors are
    bitwise equal; and they match the oracle's update_svd."""
    import paratime_b200 as B
    from oracle import paratime_np as P

    rng = np.random.default_rng(4242)
    rows, cols = 12288, 96  # 48 slabs of one 256-row TSQR leaf
    ctx = B.Context(0)
    out = {}
    base = rng.standard_normal((rows, 24))
    blocks = []
    for k in range(3):
        F = base @ rng.standard_normal((24, cols)) + 1e-3 * rng.standard_normal((rows, cols))
        G = F + 1e-2 * rng.standard_normal((rows, cols))
        blocks.append((F, G))
    for pair in ("1", "0"):
        monkeypatch.setenv("PTB_QR2_PAIR", pair)
        c = B.api.Corrector(ctx)
        for F, G in blocks:
            c.update(ctx.tensor(np.ascontiguousarray(F.T)), ctx.tensor(np.ascontiguousarray(G.T)), 1e-8)
        out[pair] = c.factors()
    for a, b in zip(out["1"], out["0"]):
        assert np.array_equal(a, b)
    co = P.empty_corrector()
    for F, G in blocks:
        co = P.update_svd(co, F, G, 1e-8)
    X, S, Y = out["1"]
    assert len(S) == co.rank
    assert np.max(np.abs(S - co.S)) <= 1e-10 * co.S[0]
    # Omega = X Y^T (procrustes.cpp:82-86) as an operator: individual vectors of clustered singular
    # values are not comparable, the product is
    V = rng.standard_normal((rows, 4))
    want = co.X @ (co.Y.T @ V)
    got = X @ (Y.T @ V)
    assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)  # noise-level directions are kept (tol 1e-8)
    F, G = blocks[-1]
    c = B.api.Corrector(ctx)
    for Fb, Gb in blocks:
        c.update(ctx.tensor(np.ascontiguousarray(Fb.T)), ctx.tensor(np.ascontiguousarray(Gb.T)), 1e-8)
    res = c.residual(ctx.tensor(np.ascontiguousarray(F.T)), ctx.tensor(np.ascontiguousarray(G.T)))
    assert res == pytest.approx(P.relative_residual(co, F, G), rel=1e-6)
