"""Workload for one ncu pass over every kernel of an LM iteration (not a bench):
linearize + damp, a 2-term series, back-substitution, trial cost, on a config.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active \
        --clock-control none -k regex:'k_(lin|cam|damp|wt|cost|sum|term|lm)' --csv --log-file out.csv \
        python tools/prof_all.py c5 1.0
    python tools/kernels_md.py out.csv c5 > profiles/<tag>_kernels_c5.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _cfg
import paper_2204_12834_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
p = _cfg.load(name, scale)
for it in range(2):  # the second pass is the warm one
    s = P.assemble(p, lam=1e-4)
    r = P.power_series_solve(s, 1e-300, 2)
    dl = P.back_substitute(s, r.delta_p)
    c, _ = P.residual_cost(p, P.BaState.from_problem(p))
print("ok", p.n_observations, r.order_used, c)
