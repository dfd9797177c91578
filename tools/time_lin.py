"""Median wall time of one device-resident relinearization (for library A/B runs).

    POBA_LIB=libab/<variant>/libpoba.so python tools/time_lin.py c5 1.0 [tag]
"""
import os
import sys
import time

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
ts = []
for _ in range(12):
    t = time.perf_counter()
    dev.linearize(p.camera_params)
    ts.append(time.perf_counter() - t)
import hashlib
from paper_2204_12834_b200 import _lib
u0, bp = dev.read(_lib.READ_U0), dev.read(_lib.READ_B_P)
h = hashlib.blake2b(np.ascontiguousarray(u0).tobytes() + np.ascontiguousarray(bp).tobytes(), digest_size=8).hexdigest()
print(f"{name} x{scale} {tag} fp{prec}: linearize {1e3 * np.median(ts[2:]):.3f} ms (median of 10), |U0| "
      f"{np.linalg.norm(u0):.17g}, U0/b_p hash {h}")
