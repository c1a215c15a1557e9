"""Host-only C++ suites on the drop-in API (no GPU needed: plain text I/O):
tests/refsuite/test_checkpoint.cpp (PhaseCorrector::save/load, procrustes.hpp:41-43) and
tests/refsuite/test_speed_model.cpp (speed-model file ingestion, experiment.hpp:86-90), built
against include/paratime/*.hpp and libparatime_b200.so."""
import shutil
import subprocess
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent / "refsuite"
LIB = Path(__file__).resolve().parent.parent / "paratime_b200" / "libparatime_b200.so"


@pytest.mark.parametrize("suite", ["test_checkpoint", "test_speed_model"])
def test_host_suite(suite):
    if not LIB.exists():
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    if shutil.which("g++") is None or shutil.which("make") is None:
        pytest.skip("no host C++ toolchain")
    subprocess.run(["make", "-s", "-C", str(HERE), "own"], check=True)
    r = subprocess.run([str(HERE / "_bin" / suite)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed checks: 0" in r.stdout
