"""Run-record CSV schemas of the reference's harness (experiment.cpp:596-628, write_run_files:
errors.csv, residuals.csv, summary.csv) on the drop-in API (include/paratime/run_files.hpp,
ptb_run_csv): byte-equal to the files the reference itself wrote for the same run records.
Pinned by tests/golden/run_csv_fixtures.json (made by the reference's run_experiment,
tests/golden/make_runfiles_golden.py).  Host-only: no GPU needed."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import paratime_b200 as B

FIX = json.loads((Path(__file__).resolve().parent / "golden" / "run_csv_fixtures.json").read_text())


def _records(files):
    rows = [r.split(",") for r in files["errors"].splitlines()[1:]]
    K = max(int(r[0]) for r in rows) + 1
    N1 = max(int(r[1]) for r in rows) + 1
    ee = np.full((K, N1), np.nan)
    l2 = np.full((K, N1), np.nan)
    for r in rows:
        ee[int(r[0]), int(r[1])] = float(r[2])
        l2[int(r[0]), int(r[1])] = float(r[3])
    res = np.full(K, math.nan)
    rank = np.zeros(K, dtype=np.int32)
    for r in files["residuals"].splitlines()[1:]:
        k, v, rk = r.split(",")
        res[int(k)] = float(v)
        rank[int(k)] = int(rk)
    div = np.zeros(K, dtype=np.int32)
    for r in files["summary"].splitlines()[1:]:
        f = r.split(",")
        div[int(f[0])] = int(f[3])
    return ee, l2, res, rank, div


@pytest.mark.parametrize("case", FIX["cases"], ids=[c["name"] for c in FIX["cases"]])
def test_run_csv_matches_reference_bytes(case):
    ee, l2, res, rank, div = _records(case["files"])
    for which in ("errors", "residuals", "summary"):
        got = B.api.run_csv(ee, l2, res, rank, div, case["plain"], which)
        assert got == case["files"][which], which


def _g(v):  # the reference's fmt (experiment.cpp:19-23): printf "%.17g"
    return "%.17g" % v


def test_run_csv_special_values_and_diverged_flag():
    ee = np.array([[1.0, math.inf], [math.nan, 1e-300]])
    l2 = np.array([[-0.0, 2.5], [3.0, 5e-324]])
    res, rank, div = np.array([math.nan, 0.125]), np.array([0, 7]), np.array([0, 1])
    want = "iteration,coupling,energy_error,l2_error,diverged\n" + "".join(
        f"{k},{n},{_g(ee[k, n])},{_g(l2[k, n])},{div[k]}\n" for k in range(2) for n in range(2))
    assert B.api.run_csv(ee, l2, res, rank, div, False, "errors") == want
    assert B.api.run_csv(ee, l2, res, rank, div, False, "residuals") == "iteration,residual,rank\n1,0.125,7\n"
    assert B.api.run_csv(ee, l2, res, rank, div, True, "residuals") == "iteration,residual,rank\n"
    assert B.api.run_csv(ee, l2, res, rank, div, False, "summary") == "iteration,energy_error,l2_error,diverged\n" + (
        f"0,{_g(math.inf)},2.5,0\n1,{_g(1e-300)},{_g(5e-324)},1\n")
