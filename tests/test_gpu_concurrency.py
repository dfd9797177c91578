"""Concurrent use of one problem's device context.

The reference's evalkit.run_benchmark(parallel=True) (evalkit.py:162-196) runs
every solver spec on the same problem in a thread pool; with the drop-in
patches those runs share the problem's libpoba context.  Each run holds the
context's lock (blocks.DeviceProblem.lock), so the traces must equal the
sequential ones exactly, and interleaved standalone calls (linearize / damp /
solve / back-substitute from two threads) must equal their sequential results.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import golden_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2204_12834_b200 as pkg
    return pkg


def test_parallel_lm_runs_match_sequential(P):
    p, _ = golden_problem("c2")
    specs = [P.LmConfig(solver="poba", max_outer_iterations=8, max_order=32),
             P.LmConfig(solver="pcg", max_outer_iterations=8),
             P.LmConfig(solver="poba", max_outer_iterations=8, max_order=10, precision=32)]
    seq = [[i.cost for i in P.run(p, c).iterations] for c in specs]
    for _ in range(3):
        with ThreadPoolExecutor(max_workers=len(specs)) as ex:
            par = list(ex.map(lambda c: [i.cost for i in P.run(p, c).iterations], specs))
        assert par == seq


def test_interleaved_systems_match_sequential(P):
    p, _ = golden_problem("c2")
    rng = np.random.default_rng(5)
    states = [P.BaState(p.camera_params.copy(), p.points + rng.normal(0, 0.01, p.points.shape)) for _ in range(4)]

    def solve(st_lam):
        st, lam = st_lam
        s = P.assemble(p, st, lam=lam)
        r = P.power_series_solve(s, 0.01, 20)
        dl = P.back_substitute(s, r.delta_p)
        c, _ = P.residual_cost(p, st)
        return r.delta_p, r.order_used, dl, c

    work = [(st, lam) for st in states for lam in (1e-4, 1e-2)]
    seq = [solve(w) for w in work]
    with ThreadPoolExecutor(max_workers=4) as ex:
        par = list(ex.map(solve, work))
    for a, b in zip(seq, par):
        assert np.array_equal(a[0], b[0]) and a[1] == b[1] and np.array_equal(a[2], b[2]) and a[3] == b[3]
