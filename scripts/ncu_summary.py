"""Summarise ncu outputs into profiles/ (tracked).

  python scripts/ncu_summary.py ROUND LAUNCH_CSV FULL_REP --grid 2048 --batch 64 --mode fast --plan "..."

* LAUNCH_CSV: `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file` output
  -> profiles/rNN_launches.md (per-kernel count, total/mean time, share of the profiled time).
* FULL_REP: `ncu --set full` report of one launch of the dominant kernel
  -> profiles/rNN_k1_full.md (headline metrics) and profiles/k1_ncu.json (DRAM bytes per launch,
  read by bench.py to fill roofline.traffic when grid/batch/mode/plan match).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def launches(path: Path):
    text = path.read_text()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    unit = rows[0]["Metric Unit"] if rows else ""
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"]
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v[1] for v in agg.values())
    return agg, total, unit, len(rows)


def raw_metrics(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (u[i], v[i]) for i, k in enumerate(h)}


def num(m, k):
    unit, val = m[k]
    x = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
    return x * scale


def launches_only(argv):
    """python scripts/ncu_summary.py launches NAME LAUNCH_CSV "command" -> profiles/NAME.md"""
    name, path, command = argv[0], Path(argv[1]), argv[2]
    agg, total, unit, n = launches(path)
    lines = [f"# {name}: ncu launch list", "", f"Command: `{command}`", "",
             f"`ncu --metrics gpu__time_duration.sum --clock-control none` — {n} launches, "
             f"{total / 1e6:.1f} ms of kernel time (serialised, cold-cache: compare shares).", "",
             f"| kernel | launches | total ({unit}) | mean ({unit}) | share |", "|---|---:|---:|---:|---:|"]
    for kname, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        short = kname if len(kname) < 90 else kname[:87] + "..."
        lines.append(f"| `{short}` | {cnt} | {t:.1f} | {t / cnt:.1f} | {100 * t / total:.1f}% |")
    out = ROOT / "profiles" / f"{name}.md"
    out.write_text("\n".join(lines) + "\n")
    print(out.read_text())


def main():
    import sys

    if len(sys.argv) > 1 and sys.argv[1] == "launches":
        launches_only(sys.argv[2:])
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("round", type=int)
    ap.add_argument("launch_csv", type=Path)
    ap.add_argument("full_rep", type=Path)
    ap.add_argument("--grid", type=int, required=True)
    ap.add_argument("--batch", type=int, required=True)
    ap.add_argument("--mode", required=True)
    ap.add_argument("--plan", required=True)
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    tag = f"r{a.round:02d}"

    agg, total, unit, n = launches(a.launch_csv)
    lines = [f"# {tag}: ncu launch list", "", f"Command: `{a.command}`", "",
             f"`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` — {n} launches profiled "
             f"(serialised, cold-cache: compare shares, not absolute times).", "",
             f"| kernel | launches | total ({unit}) | mean ({unit}) | share |", "|---|---:|---:|---:|---:|"]
    for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        short = name if len(name) < 90 else name[:87] + "..."
        lines.append(f"| `{short}` | {cnt} | {t:.1f} | {t / cnt:.1f} | {100 * t / total:.1f}% |")
    (prof / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")

    m = raw_metrics(a.full_rep)
    dur = num(m, "gpu__time_duration.sum")
    rd, wr = num(m, "dram__bytes_read.sum"), num(m, "dram__bytes_write.sum")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__block_size", "launch__grid_size", "launch__occupancy_limit_registers",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    stalls = sorted(((k, num(m, k)) for k in m if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not k.endswith("_not_issued")), key=lambda x: -x[1])
    tot = sum(v for _, v in stalls) or 1.0
    kname = max(agg.items(), key=lambda x: x[1][1])[0] if agg else m.get("Kernel Name", ("", "?"))[1]
    md = [f"# {tag}: `ncu --set full` of the dominant kernel", "", f"Kernel: `{kname}`  ", f"Plan: `{a.plan}`  ",
          f"Workload: grid {a.grid}^2, {a.batch} slices, {a.mode} mode", "", "| metric | unit | value |",
          "|---|---|---:|"]
    for k in keys:
        if k in m:
            md.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    md += ["", f"DRAM bytes per launch: {rd + wr:.4g} (read {rd:.4g}, write {wr:.4g}); algorithmic "
                f"{a.batch * a.grid * a.grid * 40:.4g} (u, udot, coef read + u, udot written, 8 B each).", "",
           "Warp-stall samples (share):", ""]
    md += [f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * v / tot:.1f}%" for k, v in stalls[:10]]
    (prof / f"{tag}_k1_full.md").write_text("\n".join(md) + "\n")
    (prof / "k1_ncu.json").write_text(json.dumps({
        "grid": a.grid, "batch": a.batch, "mode": a.mode, "plan": a.plan, "kernel": kname,
        "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "duration_s": dur,
        "source": f"profiles/{tag}_k1_full.md (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"},
        indent=1) + "\n")
    print((prof / f"{tag}_launches.md").read_text())
    print("\n".join(md))


if __name__ == "__main__":
    main()
