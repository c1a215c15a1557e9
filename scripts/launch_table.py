"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
count, total ms, share.  python scripts/launch_table.py CSV [top]"""
import csv
import io
import re
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    v = v / 1e6 if u in ("nsecond", "ns") else (v / 1e3 if u in ("usecond", "us") else v)
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("ptb::<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"| `{k[:90]}` | {c} | {t:.3f} | {100 * t / tot:.1f}% |")
print(f"| total | {sum(c for c, _ in agg.values())} | {tot:.3f} | |")
