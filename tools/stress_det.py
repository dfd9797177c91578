import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "c3"; sc = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
p = configs.make_config(name, sc)
s = P.assemble(p, lam=1e-4)
ref = P.power_series_solve(s, 1e-300, 16).delta_p
bad = 0
for k in range(30):
    d = P.power_series_solve(s, 1e-300, 16).delta_p
    if not np.array_equal(d, ref):
        bad += 1
        print("mismatch", k, np.abs(d - ref).max() / np.abs(ref).max())
print(name, sc, "mismatches", bad, "of 30")
