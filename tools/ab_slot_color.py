"""A/B of the bank-aware accumulator slot numbering (store.cu color_chunk_slots).

    python tools/ab_slot_color.py [config] [scale]

Builds the same problem twice (POBA_NO_SLOT_COLOR set / unset), times the
fused term kernel with CUDA events inside the library, and checks that the
series solution is bitwise identical (only the slot numbering differs).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2204_12834_b200 import blocks, configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
p = configs.make_config(name, scale, seed=0)
out = {}
for tag in ("first-appearance", "bank-aware", "first-appearance", "bank-aware"):
    if tag == "first-appearance":
        os.environ["POBA_NO_SLOT_COLOR"] = "1"
    else:
        os.environ.pop("POBA_NO_SLOT_COLOR", None)
    dp = blocks.DeviceProblem(p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)
    dev = dp.dev
    dev.set_points(p.points)
    dev.linearize(p.camera_params)
    dev.damp(1e-4)
    x, order, _, _ = dev.series_solve(1e-300, 16)
    ts = [dev.time_terms(20) for _ in range(3)]
    ms_term = min(t[0] for t in ts)
    ms_kernel = min(t[1] for t in ts)
    if tag in out:
        assert np.array_equal(out[tag][0], x)
    out[tag] = (x, ms_kernel)
    print(f"{name} x{scale} {tag:17s}: term kernel {ms_kernel * 1e3:8.1f} us, term {ms_term * 1e3:8.1f} us")
    dev.close()
same = np.array_equal(out["first-appearance"][0], out["bank-aware"][0])
print(f"solution bitwise identical: {same}")
