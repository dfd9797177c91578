import sys, gc
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2204_12834_b200 as P
from conftest import load_golden, golden_problem
mode = sys.argv[1] if len(sys.argv) > 1 else "lm"
if mode == "lm":
    for name, kw in [("rand3x5", {}), ("noisy4x60", {}), ("rig49", dict(max_outer_iterations=50)), ("c1", dict(max_outer_iterations=10, max_order=32)), ("c2", dict(max_outer_iterations=20, max_order=32, epsilon=1e-6))]:
        p, _ = golden_problem(name)
        tr = P.run(p, P.LmConfig(**kw))
        print(name, len(tr.iterations))
if len(sys.argv) > 2: gc.collect()
z = load_golden("explicit")
for j in range(4):
    pre = f"e{j}_"
    args = (z[pre + "cam_idx"], z[pre + "pt_idx"], z[pre + "jp"], z[pre + "jl"], z[pre + "res"], int(z[pre + "n_cam"]), int(z[pre + "n_pt"]))
    lin = P.assemble_from_observations(*args)
    s = lin.damp(float(z[pre + "lam"]))
    r, ratios = P.power_series_solve(s, 1e-14, 200, return_ratios=True)
    info = s._dp.dev.info()
    print(j, r.order_used, int(z[pre + "sys_solve0_order"]), ratios[:3], "tiles", info["n_tiles"], "work", info["n_chunks"], "partials", info["n_partials"])
