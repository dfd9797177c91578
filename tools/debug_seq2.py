import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2204_12834_b200 as P
from conftest import load_golden
z = load_golden("explicit")
for j in range(4):
    pre = f"e{j}_"
    lin = P.assemble_from_observations(z[pre + "cam_idx"], z[pre + "pt_idx"], z[pre + "jp"], z[pre + "jl"], z[pre + "res"], int(z[pre + "n_cam"]), int(z[pre + "n_pt"]))
    s = lin.damp(float(z[pre + "lam"]))
    i = 0
    while f"{pre}sys_solve{i}_eps" in z:
        q = f"{pre}sys_solve{i}_"
        r, ratios = P.power_series_solve(s, float(z[q + "eps"]), int(z[q + "m"]), return_ratios=True)
        dl = P.back_substitute(s, r.delta_p)
        print(j, i, float(z[q + "eps"]), r.order_used, int(z[q + "order"]), ratios[:3] if ratios is not None else None)
        i += 1
