"""Bitwise repeatability of single operator passes (C3 x0.1 by default)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
sc = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
p = configs.make_config(name, sc)
s = P.assemble(p, lam=1e-4)
s._activate()
dev = s._dp.dev
rng = np.random.default_rng(1)
for op in (_lib.OP_WVW, _lib.OP_W, _lib.OP_SCHUR):
    nin = 3 * p.n_points if op == _lib.OP_W else 9 * p.n_cameras
    v = rng.standard_normal(nin)
    ref = dev.apply(op, v)
    bad = []
    for k in range(reps):
        o = dev.apply(op, v)
        if not np.array_equal(o, ref):
            d = np.nonzero(o != ref)[0]
            bad.append((k, len(d), float(np.abs(o - ref).max() / np.abs(ref).max()), d[:5].tolist()))
    print("op", op, "mismatching reps", len(bad), "of", reps, bad[:5], flush=True)
