"""Drive every device entry point once on a small problem -- the workload for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py mixed
    (names: mixed, c1, c2, or cN:scale, e.g. c3:0.1)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import _lib, configs

name = sys.argv[1] if len(sys.argv) > 1 else "mixed"
if name == "mixed":
    p = configs.make_mixed_tracks()
elif ":" in name:
    n, s = name.split(":")
    p = configs.make_config(n, float(s), seed=0)
else:
    p = configs.make_config(name, 1.0, seed=0)
for prec in (64, 32):
    lin = P.linearize(p, precision=prec)
    s = lin.damp(1e-4)
    r = P.power_series_solve(s, 1e-300, 6)
    dl = P.back_substitute(s, r.delta_p)
    v = np.random.default_rng(0).standard_normal(9 * p.n_cameras)
    for op in (_lib.OP_W, _lib.OP_WT, _lib.OP_WVW, _lib.OP_SCHUR, _lib.OP_U_INV, _lib.OP_V_INV):
        x = v if op in (_lib.OP_WT, _lib.OP_WVW, _lib.OP_SCHUR, _lib.OP_U_INV) else np.ones(3 * p.n_points)
        s._op(op, x)
    P.pcg_schur_jacobi(s, max_iter=5)
    P.residual_cost(p, P.BaState.from_problem(p))
tr = P.run(p, P.LmConfig(max_outer_iterations=3, max_order=8))
print(f"sanitize workload ok: {name}, {p.n_observations} obs, final cost {tr.final_cost:.6g}")
