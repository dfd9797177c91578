"""A/B of the accumulator slot numbering (store.cu color_chunk_slots).

    python tools/ab_slot_color.py [config] [scale] [variants...]

variants: none (first-appearance numbering, POBA_NO_SLOT_COLOR), g8 / g16 /
g32 (bank-aware colouring over groups of 8 / 16 / 32 lanes), p0 / p4 / p8
(greedy colouring followed by 0 / 4 / 8 local-search passes).  With
POBA_SLOT_STATS=1 the library prints its bank-conflict model per build.  Builds the same
problem once per variant (interleaved twice), times the fused term kernel
with CUDA events inside the library, and checks that the series solution is
bitwise identical across variants (only the slot numbering differs).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2204_12834_b200 import blocks, configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
variants = sys.argv[3:] or ["none", "g32"]
p = configs.make_config(name, scale, seed=0)
out = {}
for tag in variants * 2:
    for k in ("POBA_NO_SLOT_COLOR", "POBA_SLOT_GROUP", "POBA_SLOT_PASSES"):
        os.environ.pop(k, None)
    if tag == "none":
        os.environ["POBA_NO_SLOT_COLOR"] = "1"
    elif tag.startswith("g"):
        os.environ["POBA_SLOT_GROUP"] = tag[1:]
    elif tag.startswith("p"):
        os.environ["POBA_SLOT_PASSES"] = tag[1:]
    dp = blocks.DeviceProblem(p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)
    dev = dp.dev
    dev.set_points(p.points)
    dev.linearize(p.camera_params)
    dev.damp(1e-4)
    x, order, _, _ = dev.series_solve(1e-300, 16)
    ts = [dev.time_terms(30) for _ in range(5)]
    ms_term = float(np.median([t[0] for t in ts]))
    ms_kernel = float(np.median([t[1] for t in ts]))
    if tag in out:
        assert np.array_equal(out[tag][0], x)
    out[tag] = (x, ms_kernel)
    print(f"{name} x{scale} {tag:5s}: term kernel {ms_kernel * 1e3:8.1f} us, term {ms_term * 1e3:8.1f} us (median of 5x30)")
    dev.close()
xs = [v[0] for v in out.values()]
print(f"solution bitwise identical across variants: {all(np.array_equal(xs[0], x) for x in xs)}")
