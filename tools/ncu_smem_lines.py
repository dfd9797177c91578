"""Shared-memory wavefronts per SASS instruction of an ncu report (source page):
    python tools/ncu_smem_lines.py rep.ncu-rep [n_tiles]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: h.index(k) for k in ("Source", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "Instructions Executed")}
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
items = []
for r in rows[2:]:
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
    except ValueError:
        continue
    if wf > 0:
        items.append((wf, float(r[ix["L1 Wavefronts Shared Ideal"]] or 0), r[ix["Source"]].strip()))
tot = sum(w for w, _, _ in items)
print(f"total shared wavefronts {tot / 1e6:.1f} M ({tot / per:.1f} per tile)")
groups = {}
for wf, ideal, src in items:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    g = groups.setdefault(op, [0, 0.0, 0.0])
    g[0] += 1
    g[1] += wf
    g[2] += ideal
for op, (n, wf, ideal) in sorted(groups.items(), key=lambda x: -x[1][1]):
    print(f"  {op:28s} x{n:3d}  {wf / per:7.1f} per tile  (ideal {ideal / per:6.1f})")
