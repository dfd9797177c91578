import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs
from oracle import poba_oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
p = configs.make_config(name, scale)
lin = P.linearize(p)
print(lin._dp.dev.info())
U0g, bpg, V0g = lin.U0, lin.b_p, lin.V0
t = time.time()
lo = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
print("oracle lin %.1fs" % (time.time() - t), "invalid", lo.n_invalid, lin.n_invalid)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
print("U0 rel", rel(U0g, lo.U0), "bp rel", rel(bpg, lo.b_p), "V0 rel", rel(V0g, lo.V0), "bl rel", rel(lin.b_l, lo.b_l))
bad = np.flatnonzero(np.abs(U0g - lo.U0).reshape(len(U0g), -1).max(1) > 1e-9 * np.abs(lo.U0).reshape(len(U0g), -1).max(1))
print("bad cams", bad[:20], len(bad))
try:
    so = O.OracleSystem(lo, 1e-4); print("oracle damp ok")
except Exception as e: print("oracle damp:", e)
