"""Minimal workload for ncu: C5 assemble, one series solve, back-substitution twice."""
import sys
sys.path.insert(0, ".")
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs
p = configs.make_config(sys.argv[1] if len(sys.argv) > 1 else "c5", float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
s = P.assemble(p, lam=1e-4)
r = P.power_series_solve(s, 1e-2, 32)
for _ in range(2):
    P.back_substitute(s, r.delta_p)
print("ok")
