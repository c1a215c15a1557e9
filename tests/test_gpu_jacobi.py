"""The multi-CTA Jacobi SVD (k_jacobi_coop, used when H does not fit one CTA's shared memory)
must reproduce the single-CTA kernel bitwise and be an accurate SVD (procrustes.cpp:58,220
BDCSVD, pinned by test_procrustes.cpp's dense-SVD oracle at 1e-10)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _run(p, q, path, jacobi):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    if jacobi:
        env["PTB_JACOBI"] = jacobi
    subprocess.run([sys.executable, str(ROOT / "tests" / "svd_probe.py"), str(p), str(q), str(path)], check=True,
                   env=env, timeout=600)
    return np.load(path)


@pytest.mark.parametrize("shape", [(300, 290), (290, 300), (420, 180)])
def test_coop_jacobi_matches_single_cta_bitwise(tmp_path, shape):
    p, q = shape
    a = _run(p, q, tmp_path / "coop.npz", "coop")
    b = _run(p, q, tmp_path / "single.npz", "single")
    for key in ("U", "S", "V"):
        assert np.array_equal(a[key], b[key]), key
    m, U, S, V = a["m"], a["U"], a["S"], a["V"]
    ref = np.linalg.svd(m, compute_uv=False)
    assert np.max(np.abs(S - ref) / ref[0]) <= 1e-13
    assert np.linalg.norm(m - (U * S) @ V.T) <= 1e-12 * np.linalg.norm(m)  # reference pins 1e-12 (planted)
    k = min(p, q)
    assert np.max(np.abs(V.T @ V - np.eye(k))) <= 1e-12


@pytest.mark.parametrize("path", ["auto", "small"])
@pytest.mark.parametrize("shape", [(108, 108), (60, 44), (44, 60), (33, 33), (7, 5), (150, 120), (250, 240)])
def test_small_and_cluster_jacobi_are_accurate(tmp_path, shape, path):
    """k_jacobi_cluster (default from 24 columns: rows split over a thread-block cluster) and
    k_jacobi_small (one CTA's shared memory) on the corrector's H sizes at cfg1-3."""
    p, q = shape
    a = _run(p, q, tmp_path / "small.npz", None if path == "auto" else path)  # auto: cluster from 64 columns
    m, U, S, V = a["m"], a["U"], a["S"], a["V"]
    ref = np.linalg.svd(m, compute_uv=False)
    assert np.max(np.abs(S - ref) / ref[0]) <= 1e-13
    assert np.linalg.norm(m - (U * S) @ V.T) <= 1e-12 * np.linalg.norm(m)
    k = min(p, q)
    assert np.max(np.abs(V.T @ V - np.eye(k))) <= 1e-12
    assert np.max(np.abs(U.T @ U - np.eye(k))) <= 1e-12
