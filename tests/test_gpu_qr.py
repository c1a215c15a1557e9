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
