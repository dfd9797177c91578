"""Where the end-to-end step's time goes (C5 by default): assemble / solve / back-substitution."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = configs.make_config(name, 1.0)
st = configs.LM_SETTINGS[name]
cams = torch.from_numpy(p.camera_params).pin_memory().numpy()
pts = torch.from_numpy(p.points).pin_memory().numpy()


class S:
    camera_params = cams
    points = pts


for _ in range(2):
    s = P.assemble(p, S, lam=st.initial_lambda)
    r = P.power_series_solve(s, st.epsilon, st.max_order)
    P.back_substitute(s, r.delta_p)
dev = s._dp.dev
T = {"linearize": [], "damp": [], "solve": [], "back_sub": [], "total": []}
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lin = P.linearize(p, S)
    t1 = time.perf_counter()
    s = lin.damp(st.initial_lambda)
    s._activate()
    t2 = time.perf_counter()
    r = P.power_series_solve(s, st.epsilon, st.max_order)
    t3 = time.perf_counter()
    dl = P.back_substitute(s, r.delta_p)
    t4 = time.perf_counter()
    for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
        T[k].append(1e3 * v)
print(name, {k: f"{np.median(v):.2f} ms" for k, v in T.items()}, "order", r.order_used)
# device-only parts
t = time.perf_counter(); dev.set_points(pts); torch.cuda.synchronize(); print("set_points", 1e3 * (time.perf_counter() - t))
t = time.perf_counter(); dev.linearize(cams); print("dev.linearize(cams)", 1e3 * (time.perf_counter() - t))
t = time.perf_counter(); dev.damp(st.initial_lambda); print("dev.damp", 1e3 * (time.perf_counter() - t))
t = time.perf_counter(); dev.series_solve(st.epsilon, st.max_order); print("dev.series_solve", 1e3 * (time.perf_counter() - t))
t = time.perf_counter(); dev.back_substitute(None); print("dev.back_substitute(None)+D2H", 1e3 * (time.perf_counter() - t))
t = time.perf_counter(); dev.back_substitute(None, want_delta_l=False); print("dev.back_substitute no D2H", 1e3 * (time.perf_counter() - t))
