"""PhaseCorrector::save/load on the drop-in C++ API (procrustes.hpp:41-43), host-only.

Builds tests/refsuite/test_checkpoint.cpp against include/paratime/*.hpp and
libparatime_b200.so (no GPU needed: the checkpoint is plain text I/O) and runs it."""
import shutil
import subprocess
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent / "refsuite"
LIB = Path(__file__).resolve().parent.parent / "paratime_b200" / "libparatime_b200.so"


def test_checkpoint_suite():
    if not LIB.exists():
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    if shutil.which("g++") is None or shutil.which("make") is None:
        pytest.skip("no host C++ toolchain")
    subprocess.run(["make", "-s", "-C", str(HERE), "own"], check=True)
    r = subprocess.run([str(HERE / "_bin" / "test_checkpoint")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed checks: 0" in r.stdout
