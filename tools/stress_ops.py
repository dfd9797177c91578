import sys, gc
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2204_12834_b200 as P
from conftest import golden_problem
from oracle import poba_oracle as O
p, _ = golden_problem("noisy4x60")
lin_o = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
so = O.OracleSystem(lin_o, 1e-2)
rng = np.random.default_rng(0)
v = rng.normal(size=3 * p.n_points)
want = so.apply_w(v)
bad = 0
for k in range(60):
    q = p.copy()  # fresh arrays -> fresh device context each time
    s = P.assemble(q, lam=1e-2)
    got = s.apply_w(v)
    r = np.linalg.norm(got - want) / np.linalg.norm(want)
    if r > 1e-12:
        bad += 1
        print("bad", k, r)
    del s, q
    if k % 7 == 0: gc.collect()
print("bad", bad, "of 60")
