"""Device timeline of one end-to-end step (assemble -> solve -> back-substitution) via CUPTI.

    python tools/trace_e2e.py [config] [scale]

Uses torch.profiler (kineto/CUPTI) only as a tracer: it records every kernel
and copy the library issues, with device timestamps, so the step's wall time
can be split into kernels, copies and gaps.  Not a bench number.
"""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
import _cfg
p = _cfg.load(name, scale)
st = configs.LM_SETTINGS.get(name, configs.LmSettings())
cams = torch.from_numpy(p.camera_params).pin_memory().numpy()
pts = torch.from_numpy(p.points).pin_memory().numpy()


class S:
    camera_params = cams
    points = pts


def step():
    marks = [time.perf_counter()]
    s = P.assemble(p, S, lam=st.initial_lambda)
    s._activate()
    marks.append(time.perf_counter())
    r = P.power_series_solve(s, st.epsilon, st.max_order)
    marks.append(time.perf_counter())
    P.back_substitute(s, r.delta_p)
    marks.append(time.perf_counter())
    return marks


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    marks = step()
    torch.cuda.synchronize()
print(f"{name} x{scale}: wall assemble {1e3 * (marks[1] - marks[0]):.2f} ms, solve {1e3 * (marks[2] - marks[1]):.2f} ms, "
      f"back-sub {1e3 * (marks[3] - marks[2]):.2f} ms")
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
agg = defaultdict(lambda: [0, 0.0])
for e in evs:
    k = e.name[:70]
    agg[k][0] += 1
    agg[k][1] += e.time_range.elapsed_us()
tot = sum(v[1] for v in agg.values())
print(f"{len(evs)} device activities, {tot / 1e3:.2f} ms busy (sum of durations)")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {us / 1e3:8.3f} ms  x{n:4d}  {k}")
if evs:
    t0 = evs[0].time_range.start
    t1 = max(e.time_range.end for e in evs)
    print(f"device span {1e-3 * (t1 - t0):.2f} ms")
    gaps = []
    end = evs[0].time_range.end
    for a in evs[1:]:
        if a.time_range.start > end + 50:
            gaps.append((a.time_range.start - end, a.name[:50], 1e-3 * (end - t0)))
        end = max(end, a.time_range.end)
    gaps.sort(reverse=True)
    print("largest idle gaps (us, next activity, at ms):")
    for g in gaps[:12]:
        print(f"  {g[0]:8.0f}  {g[1]}  @{g[2]:.2f}")
