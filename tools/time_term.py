"""Median device time of the fused series term on a config (for library A/B runs).

    POBA_LIB=libab/<variant>/libpoba.so python tools/time_term.py c5 1.0 [tag]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2204_12834_b200 import blocks, configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tag = sys.argv[3] if len(sys.argv) > 3 else os.environ.get("POBA_LIB", "default")
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 64
import _cfg
p = _cfg.load(name, scale)
dp = blocks.DeviceProblem(p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)
dev = dp.dev
dev.set_points(p.points)
dev.set_precision(prec)
dev.linearize(p.camera_params)
dev.damp(1e-4)
try:
    x, order, _, _ = dev.series_solve(1e-300, 16)
except Exception as e:  # ablation builds (tools only) may produce vanishing / non-finite iterates
    print("series_solve:", e)
    x = np.zeros(1)
ts = [dev.time_terms(20) for _ in range(5)]
print(f"{name} x{scale} {tag} fp{prec}: term kernel {1e3 * np.median([t[1] for t in ts]):8.1f} us, "
      f"term {1e3 * np.median([t[0] for t in ts]):8.1f} us, |x| {np.linalg.norm(x):.17g}")
