"""Where a bench step's time goes: device kernels vs gaps for dev.series_solve
on a config (CUPTI trace through torch.profiler; a diagnostic, not a bench number).

    python tools/step_gaps.py [config] [scale] [steps]
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2204_12834_b200 import blocks, configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = configs.make_config(name, scale, seed=0)
st = configs.LM_SETTINGS.get(name, configs.LmSettings())
dp = blocks.DeviceProblem(p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)
dev = dp.dev
dev.set_points(p.points)
dev.linearize(p.camera_params)
dev.damp(st.initial_lambda)
for _ in range(5):
    dev.series_solve(st.epsilon, st.max_order)
torch.cuda.synchronize()
stream = torch.cuda.ExternalStream(dev.stream_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(steps):
    dev.series_solve(st.epsilon, st.max_order)
e1.record(stream)
e1.synchronize()
print(f"untraced: {e0.elapsed_time(e1) / steps:.3f} ms per step")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        dev.series_solve(st.epsilon, st.max_order)
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
span = (evs[-1].time_range.end - evs[0].time_range.start) / 1e3
busy = sum(e.time_range.end - e.time_range.start for e in evs) / 1e3
agg = defaultdict(lambda: [0, 0.0])
for e in evs:
    agg[e.name[:60]][0] += 1
    agg[e.name[:60]][1] += (e.time_range.end - e.time_range.start) / 1e3
print(f"traced: span {span / steps:.3f} ms per step, busy {busy / steps:.3f} ms per step")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
    print(f"  {t / steps:8.3f} ms/step  x{n / steps:5.1f}  {k}")
gaps = sorted(((evs[i + 1].time_range.start - evs[i].time_range.end) / 1e3, evs[i + 1].name[:50])
              for i in range(len(evs) - 1))[::-1][:8]
print("largest gaps (ms):", [(round(g, 3), n) for g, n in gaps])
