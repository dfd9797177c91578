import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2204_12834_b200 import _lib, configs
p = configs.make_config("c5", 1.0)
dev = _lib.Device(0)
for i in range(2):
    t = time.perf_counter(); dev.set_problem(p.n_cameras, p.n_points, p.cam_indices, p.pt_indices, p.pixels); print("set_problem", time.perf_counter() - t)
t = time.perf_counter(); dev.set_points(p.points); dev.linearize(p.camera_params); print("linearize", time.perf_counter() - t)
t = time.perf_counter(); o = dev.ordering(); print("ordering export", time.perf_counter() - t)
