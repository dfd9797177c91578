import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2204_12834_b200 as P
from conftest import load_golden
from oracle import poba_oracle as O
z = load_golden("explicit")
for j in range(4):
    pre = f"e{j}_"
    args = (z[pre + "cam_idx"], z[pre + "pt_idx"], z[pre + "jp"], z[pre + "jl"], z[pre + "res"], int(z[pre + "n_cam"]), int(z[pre + "n_pt"]))
    lin = P.assemble_from_observations(*args)
    s = lin.damp(float(z[pre + "lam"]))
    lo = O.linearize_explicit(*args); so = O.OracleSystem(lo, float(z[pre + "lam"]))
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    print(j, "ncam", args[5], "npt", args[6], "nobs", len(args[0]), "bt", rel(s.b_tilde(), so.b_tilde()), s._dp.dev.info()["n_tiles"], s._dp.dev.info()["k_max"])
    for m in (0, 1, 2, 3):
        g = P.power_series_solve(s, 1e-300, m).delta_p
        w, _, _ = O.series_solve(so, 1e-300, m)
        print("   m", m, rel(g, w))
print("---- eps 1e-14 solves, repeated")
for j in range(4):
    pre = f"e{j}_"
    args = (z[pre + "cam_idx"], z[pre + "pt_idx"], z[pre + "jp"], z[pre + "jl"], z[pre + "res"], int(z[pre + "n_cam"]), int(z[pre + "n_pt"]))
    lin = P.assemble_from_observations(*args)
    s = lin.damp(float(z[pre + "lam"]))
    for rep in range(3):
        r, ratios = P.power_series_solve(s, 1e-14, 200, return_ratios=True)
        print(j, rep, r.order_used, r.converged, ratios[:4], "golden order", int(z[pre + "sys_solve0_order"]))
