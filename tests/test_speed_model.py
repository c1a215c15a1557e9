"""Speed-model text format (experiment.hpp:84-90, experiment.cpp:711-784) on the B200 library's
host API: writer byte-equal to the reference's, reader values exact, the reference's ConfigError
cases and messages.  Pinned by tests/golden/speed_model_fixtures.json (made by the reference
itself, tests/golden/make_speed_golden.py); where oracle/_ref is built, also against the live
reference on random fields.  Host-only: no GPU needed."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paratime_b200 as B

HERE = Path(__file__).resolve().parent
FIX = json.loads((HERE / "golden" / "speed_model_fixtures.json").read_text())
TOOL = HERE.parent / "oracle" / "_ref" / "speed_model_tool"


def _grid(f):
    if f["dim"] == 1:
        return B.Grid((f["n"][0],), (f["h"][0],))
    return B.Grid(tuple(f["n"]), tuple(f["h"]))


@pytest.mark.parametrize("i", range(len(FIX["fields"])))
def test_writer_matches_reference_bytes(i):
    f = FIX["fields"][i]
    assert B.api.write_speed_model(_grid(f), np.array(f["c"])) == f["text"]


@pytest.mark.parametrize("i", range(len(FIX["fields"])))
def test_reader_reads_reference_text_exactly(i):
    f = FIX["fields"][i]
    g, c = B.api.read_speed_model(f["text"])
    assert g.n == _grid(f).n and g.h == _grid(f).h
    assert np.array_equal(c.ravel(), np.array(f["c"]))


@pytest.mark.parametrize("i", range(len(FIX["bad"])))
def test_malformed_input_raises_config_error_like_reference(i):
    b = FIX["bad"][i]
    assert b["code"] == 5
    with pytest.raises(B.PtbError) as e:
        B.api.read_speed_model(b["text"])
    assert e.value.status == B.api.CONFIG
    assert b["out"] == "CONFIG_ERROR " + str(e.value).split("] ", 1)[1]


@pytest.mark.skipif(not TOOL.exists(), reason="oracle/_ref not built")
def test_random_fields_against_live_reference():
    rng = np.random.default_rng(11)
    for _ in range(20):
        if rng.random() < 0.3:
            dim, n0, n1 = 1, int(rng.integers(4, 40)), 1
            h0, h1 = float(rng.uniform(0.01, 1)), 1.0
            g = B.Grid((n0,), (h0,))
        else:
            dim, n0, n1 = 2, int(rng.integers(4, 20)), int(rng.integers(4, 20))
            h0, h1 = float(rng.uniform(0.01, 1)), float(rng.uniform(0.01, 1))
            g = B.Grid((n0, n1), (h0, h1))
        c = np.exp(rng.standard_normal(n0 * n1) * 5)
        inp = f"{dim} {n0} {n1} {h0!r} {h1!r}\n" + " ".join(repr(float(v)) for v in c) + "\n"
        ref = subprocess.run([str(TOOL), "write"], input=inp, capture_output=True, text=True, check=True).stdout
        mine = B.api.write_speed_model(g, c)
        assert mine == ref
        _, back = B.api.read_speed_model(ref)
        assert np.array_equal(back.ravel(), c)
