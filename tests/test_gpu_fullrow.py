"""k_wave2 full-row strips (the strip spans the periodic row, no halo columns): parity with the
oracle at the FAST tolerance and bitwise coupling == repeated steps, with the planner forced to
use them (PTB_WAVE_FULL=2, read once per process -> subprocess)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_full_row_strips():
    env = dict(os.environ, PTB_WAVE_FULL="2", PYTHONPATH=str(ROOT))
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "fullrow_probe.py")], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    plans = [l for l in r.stdout.splitlines() if l.startswith("PLANS")][0]
    assert "full-row" in plans and "k_wave2<8," in plans, plans
    worst = float([l for l in r.stdout.splitlines() if l.startswith("WORST")][0].split()[1])
    assert worst <= 1e-12, worst
