"""Minimal workload for ncu: assemble a config and run a few forced series terms."""
import sys
sys.path.insert(0, ".")
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 64
import _cfg
p = _cfg.load(name, scale)
s = P.assemble(p, lam=1e-4, precision=prec)
r = P.power_series_solve(s, 1e-300, 4)
print("ok", p.n_observations, r.order_used)
