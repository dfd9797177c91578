"""Quick perf probe: generate a config, assemble on GPU, time series terms."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
precision = int(sys.argv[3]) if len(sys.argv) > 3 else 64
t = time.time(); p = configs.make_config(name, scale); tg = time.time() - t
t = time.time(); s = P.assemble(p, lam=1e-4, precision=precision); ta = time.time() - t
info = s._dp.dev.info()
r = P.power_series_solve(s, 1e-300, 8)
ms_term, ms_kernel, launches = s._dp.dev.time_terms(20)
nobs, ncam, nlm = p.n_observations, p.n_cameras, p.n_points
B = (196 if precision == 64 else 100) * nobs + 48 * nlm + 648 * ncam
print(f"{name} x{scale}: obs {nobs} cams {ncam} pts {nlm} gen {tg:.1f}s assemble {ta:.2f}s info {info}")
print(f"  term {ms_term*1e3:.1f} us (kernel {ms_kernel*1e3:.1f} us, {launches} launches) -> "
      f"{B/ms_term/1e6:.0f} GB/s overall, {B/ms_kernel/1e6:.0f} GB/s kernel (of 6540 measured)")
t = time.time(); r = P.power_series_solve(s, 1e-300, 32); t1 = time.time() - t
print(f"  solve m=32: {t1*1e3:.1f} ms wall, order {r.order_used}")
