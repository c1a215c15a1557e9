"""Run-record CSV fixtures written by the reference's own harness (experiment.cpp:596-628,
write_run_files via run_experiment), run through oracle/_ref/run_experiment_tool (built by
oracle/ref/Makefile from the reference's experiment.cpp in /root/reference).

    python tests/golden/make_runfiles_golden.py   -> tests/golden/run_csv_fixtures.json
"""
import json
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import refbind  # noqa: E402

OUT = Path(__file__).resolve().parent / "run_csv_fixtures.json"

CASES = [  # (name, preset, overrides)
    ("oned-theta", "oned-variable", "iterations=3\nvariant=theta\nworkers=1"),
    ("oned-plain", "oned-variable", "iterations=3\nvariant=plain\nworkers=1"),
    ("oned-omega-identity", "oned-variable", "iterations=2\nvariant=omega-identity\nworkers=1"),
    ("oned-corrected-coarse-only", "oned-variable", "iterations=2\nvariant=corrected-coarse-only\nworkers=1"),
    ("waveguide-theta", "waveguide", "iterations=2\nworkers=1"),
    ("no-correction", "no-correction", "iterations=2\nworkers=1"),
]


def main():
    assert refbind.build(), "needs /root/reference (oracle/_ref)"
    tool = ROOT / "oracle" / "_ref" / "run_experiment_tool"
    out = {"cases": []}
    for name, preset, ov in CASES:
        with tempfile.TemporaryDirectory() as d:
            subprocess.run([str(tool), preset, d] + ov.split("\n"), check=True, capture_output=True, timeout=600)
            files = {f: (Path(d) / f"{f}.csv").read_text() for f in ("errors", "residuals", "summary")}
        # plain parareal writes the residuals header only (experiment.cpp:613-614)
        plain = files["residuals"].count("\n") == 1
        out["cases"].append({"name": name, "preset": preset, "overrides": ov, "plain": plain, "files": files})
        print(name, len(files["errors"].splitlines()), "rows")
    OUT.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
