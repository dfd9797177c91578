"""Per-kernel table of one LM iteration from an ncu metrics CSV (tools/prof_all.py):
time, DRAM bytes, achieved GB/s (ncu DRAM traffic / duration), algorithmic bytes and
their fraction of the measured HBM peak.   python tools/kernels_md.py out.csv c5"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, idi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
SC = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "second": 1e3,
      "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    v = float(r[vi].replace(",", "")) * SC.get(r[ui], 1.0)
    per[r[idi]][r[mi]] = v
    n = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    names[r[idi]] = re.sub(r"^.*::(?=k_)", "", n)
# the workload runs the LM iteration twice: average per pass over both
PASSES = 2
agg = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(int)
for i, n in names.items():
    cnt[n] += 1
    for k, v in per[i].items():
        agg[n][k] += v
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
N = {"c5": (29084796, 4500000, 13700), "c4": (10317376, 1000000, 1100), "c3": (878990, 160000, 1200)}[cfg]
no, nl, nc = N
ALG = {  # algorithmic bytes per launch, keyed by kernel name prefix
    "k_term<0, 0": 196 * no + 48 * nl + 72 * nc, "k_term<1, 0": 196 * no + 72 * nl + 72 * nc,
    "k_lin_tile<0, 0>": (196 + 16 + 16 + 4 + 1) * no + (24 + 96) * nl,
    "k_cam_chunk_reduce<0, 0>": (16 + 4) * no + 54 * 8 * nc,
    "k_wt_tile<2, 0>": 196 * no + (48 + 24 + 24) * nl, "k_cost_tile": (16 + 4 + 1) * no + 48 * nl,
    "k_damp_v": (48 + 24 + 48 + 48) * nl, "k_damp_u": (360 + 72 + 360 + 360) * nc,
}


def alg_of(name):
    for k, v in ALG.items():
        if name.startswith(k):
            return v
    return None


peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
print(f"| kernel | launches per pass | us per pass (ncu, cold, summed over its launches) | DRAM read MB | DRAM write MB | "
      f"DRAM GB/s | algorithmic MB | algorithmic GB/s | frac of {peak:.0f} | LSU pipe % | warps active % |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
ONCE = ("k_cam_degree", "k_cam_major_gather", "k_cam_slot_keys")  # store build, not part of an iteration
for n, m in sorted(agg.items(), key=lambda x: -x[1].get("gpu__time_duration.sum", 0)):
    if n in ONCE:
        continue
    k = cnt[n]
    t = m.get("gpu__time_duration.sum", 0.0) / PASSES  # ms per pass
    rd, wr = m.get("dram__bytes_read.sum", 0.0) / PASSES, m.get("dram__bytes_write.sum", 0.0) / PASSES
    lp = k / PASSES
    alg = alg_of(n)
    if alg and n.startswith("k_term") or n.startswith("k_cam<"):
        # launched several times per pass on the same data: per-launch figures
        t, rd, wr, lp_note = t / lp, rd / lp, wr / lp, f"{lp:g} (per launch)"
    else:
        lp_note = f"{lp:g}"
    a = f"{alg / 1e6:,.0f} | {alg / t / 1e6:,.0f} | {alg / t / 1e6 / peak:.2f}" if alg else "— | — | —"
    print(f"| `{n}` | {lp_note} | {t * 1e3:,.1f} | {rd / 1e6:,.1f} | {wr / 1e6:,.1f} | {(rd + wr) / t / 1e6:,.0f} | {a} | "
          f"{m.get('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed', 0) / k:.0f} | "
          f"{m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0) / k:.0f} |")
