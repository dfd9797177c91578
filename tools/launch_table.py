"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as a markdown table.

python tools/launch_table.py launches.csv "title" > profiles/xxx.md
"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-3)
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"^poba::", "", name.split("::")[-1]) if "poba" in name else name[-60:]
    tot[name] += v * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else 'launch list'}\n")
print("Cold-cache, serialised per-launch times (ncu replays each launch); compare shares, not absolutes.\n")
print("| kernel | launches | total ms | share | mean us/launch |\n|---|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| {k} | {cnt[k]} | {tot[k]:.3f} | {100 * tot[k] / all_ms:.1f}% | {1e3 * tot[k] / cnt[k]:.1f} |")
