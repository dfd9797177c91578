"""Run-to-run bitwise repeatability of every device entry point on a small
(L2-resident) problem: each call repeated N times and compared with the first.

    python tools/det_sweep.py [config|mixed] [scale] [reps] [precision]
"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs, _lib

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
sc = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 64
p = configs.make_mixed_tracks() if name == "mixed" else configs.make_config(name, sc)
s = P.assemble(p, lam=1e-4, precision=prec)
s._activate()
dev = s._dp.dev
rng = np.random.default_rng(3)
vc = rng.standard_normal(9 * p.n_cameras)
vl = rng.standard_normal(3 * p.n_points)
cams, pts = p.camera_params, p.points
assign, ncl, _ = _lib.cluster_cameras(p.n_cameras, p.n_points, p.cam_indices, p.pt_indices, 16)


def lin():
    dev.linearize(cams, pts)
    dev.damp(1e-4)
    return np.concatenate([dev.read(k).ravel() for k in (_lib.READ_U0, _lib.READ_V0, _lib.READ_B_P,
                                                          _lib.READ_B_L, _lib.READ_D_P, _lib.READ_D_L)])


cases = {
    "linearize+damp": lin,
    "series m=12": lambda: dev.series_solve(1e-300, 12)[0],
    "series eps=1e-2": lambda: dev.series_solve(1e-2, 40)[0],
    "series_apply": lambda: dev.series_apply(vc, 6),
    "op W": lambda: dev.apply(_lib.OP_W, vl),
    "op WT": lambda: dev.apply(_lib.OP_WT, vc),
    "op WVW": lambda: dev.apply(_lib.OP_WVW, vc),
    "op SCHUR": lambda: dev.apply(_lib.OP_SCHUR, vc),
    "back_substitute": lambda: (dev.series_solve(1e-2, 20), dev.back_substitute()[0])[1],
    "cost": lambda: np.array([dev.cost(cams, pts)[0]]),
    "schur_diagonal": lambda: dev.schur_diagonal(),
    "pcg jacobi": lambda: dev.pcg(1, 0, 1e-6, 30)[0],
    "pcg series": lambda: dev.pcg(2, 3, 1e-6, 20)[0],
    "post clustered": lambda: dev.series_solve_clustered(assign, ncl, 1e-2, 20)[0],
}
fails = 0
for label, fn in cases.items():
    ref = np.array(fn(), copy=True)
    bad = 0
    for _ in range(reps):
        if not np.array_equal(np.asarray(fn()), ref):
            bad += 1
    fails += bad > 0
    print(f"{label:18s} mismatches {bad} of {reps}", flush=True)
print(name, sc, "precision", prec, "entry points with mismatches:", fails)
