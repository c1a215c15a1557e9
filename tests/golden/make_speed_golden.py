"""Speed-model text fixtures from the reference's own reader/writer (experiment.cpp:711-784),
run through oracle/_ref/speed_model_tool (built by oracle/ref/Makefile from /root/reference).

    python tests/golden/make_speed_golden.py   -> tests/golden/speed_model_fixtures.json
"""
import json
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
TOOL = ROOT / "oracle" / "_ref" / "speed_model_tool"
OUT = Path(__file__).resolve().parent / "speed_model_fixtures.json"

FIELDS = [  # (dim, n0, n1, h0, h1, seed)
    (2, 6, 5, 1 / 6, 0.2, 1),
    (1, 7, 1, 1 / 7, 1.0, 2),
    (2, 4, 4, 0.5, 0.125, 3),
    (2, 5, 8, 1 / 3, 1 / 7, 4),
]
BAD = [
    "3 junk",
    "0 4 0.1 0.1\n",
    "4 4 0.1 -0.1\n" + "1 " * 16,
    "4 4 0.1 0.1\n" + "1 " * 15,
    "4 4 0.1 0.1\n" + "1 " * 16 + "7",
    "4 4 0.1 0.1\n" + "1 " * 15 + "-2",
    "4 4 0.1 0.1\n" + "1 " * 15 + "nan",
    "3 4 0.1 0.1\n" + "1 " * 12,
    "1 3 1 0.1\n1 2 3",
    "4 2 0.1 0.1\n" + "1 " * 8,
]


def tool(mode, text):
    r = subprocess.run([str(TOOL), mode], input=text, capture_output=True, text=True)
    return r.returncode, r.stdout


def main():
    fields = []
    for dim, n0, n1, h0, h1, seed in FIELDS:
        rng = np.random.default_rng(seed)
        c = np.exp(rng.standard_normal(n0 * n1) * 4.0)  # many magnitudes: exercises %.17g
        inp = f"{dim} {n0} {n1} {h0!r} {h1!r}\n" + " ".join(repr(float(v)) for v in c) + "\n"
        code, text = tool("write", inp)
        assert code == 0, text
        fields.append({"dim": dim, "n": [n0, n1], "h": [h0, h1], "c": [float(v) for v in c], "text": text})
    bad = []
    for t in BAD:
        code, out = tool("read", t)
        bad.append({"text": t, "code": code, "out": out.strip()})
    OUT.write_text(json.dumps({"fields": fields, "bad": bad}, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
