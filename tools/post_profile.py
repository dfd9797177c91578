"""Where a PoST LM run's time goes (host clustering, second device store, per-iteration
device work):  python tools/post_profile.py [config] [scale] [max_cluster_size]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import _cfg
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import blocks, clustering, configs, lm

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
mcs = int(sys.argv[3]) if len(sys.argv) > 3 else 100
p = _cfg.load(name, scale)
st = configs.LM_SETTINGS.get(name, configs.LmSettings())
t = time.perf_counter(); dp = blocks.device_problem(p); t_store = time.perf_counter() - t
t = time.perf_counter(); part = clustering.cluster_cameras(p, mcs); t_cluster = time.perf_counter() - t
t = time.perf_counter()
cl = part.assignment[np.asarray(dp.cam_indices)]
key = np.asarray(dp.pt_indices, dtype=np.int64) * part.n_clusters + cl
uniq, virt = np.unique(key, return_inverse=True)
t_unique = time.perf_counter() - t
t = time.perf_counter(); vs = clustering._VirtualStore(dp, np.asarray(part.assignment), part.n_clusters); t_vstore = time.perf_counter() - t
print(f"{name} x{scale}: {p.n_observations} obs, {part.n_clusters} clusters (max size {mcs}), "
      f"cut observations {part.cut_observations} ({100.0 * part.cut_observations / p.n_observations:.1f}%), "
      f"virtual landmarks {len(uniq)} vs {p.n_points} landmarks")
print(f"  first device store (shared with PoBA)      {t_store:8.3f} s")
print(f"  cluster_cameras (host C++ greedy merge)    {t_cluster:8.3f} s")
print(f"  virtual-landmark keys (np.unique, host)    {t_unique:8.3f} s   (inside the next line)")
print(f"  second device store (_VirtualStore)        {t_vstore:8.3f} s")
cfg = lm.LmConfig(solver="post", max_outer_iterations=st.max_outer_iterations, epsilon=st.epsilon,
                  max_order=st.max_order, initial_lambda=st.initial_lambda, max_cluster_size=mcs)
t = time.perf_counter(); tr = lm.run(p, cfg); wall = time.perf_counter() - t
its = tr.iterations
print(f"  lm.run(solver='post') wall                 {wall:8.3f} s, {len(its) - 1} iterations, "
      f"first iteration at {its[1].cumulative_time_s if len(its) > 1 else float('nan'):.3f} s, "
      f"mean later iteration {(its[-1].cumulative_time_s - its[1].cumulative_time_s) / max(len(its) - 2, 1):.4f} s")
print(f"  cost {its[0].cost:.6g} -> {its[-1].cost:.6g}")
