"""Small determinism probe (C3 x0.1): a few solves of the same system, max relative difference."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs
m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = configs.make_config("c3", 0.1)
s = P.assemble(p, lam=1e-4)
rs = [P.power_series_solve(s, 1e-300, m).delta_p for _ in range(reps)]
print("m", m, "maxdiff", max(float(np.abs(r - rs[0]).max() / np.abs(rs[0]).max()) for r in rs[1:]))
