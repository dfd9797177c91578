"""Drop-in proof through the reference's OWN driver (INTEGRATION.md route 2).

The unmodified reference package shipped in baseline/_ref (installed by
__graft_entry__.build()) runs its own ``powerba.lm.run`` loop (lm.py:167-232)
with the hot-path functions it looks up as module globals (lm.py:16-20)
rebound to this package's GPU implementations -- linearize, the series solve,
back-substitution, the cost, memory accounting, the PCG / dense solvers.  The
traces must reproduce the reference's golden traces (tests/golden, produced by
the unpatched reference), including its criterion-6 end-to-end golden (rig49,
final cost 7584.4992), and the reference's own evaluation harness
(evalkit.run_benchmark, parallel=True: runs in a thread pool on one shared
problem) must give the same traces as its sequential mode.
"""
from __future__ import annotations

import os
import sys
import types

import numpy as np
import pytest

from conftest import REPO, golden_problem

pytestmark = pytest.mark.gpu

REF = os.path.join(REPO, "baseline", "_ref")
COST_TOL = 1e-8


@pytest.fixture(scope="module")
def patched_ref():
    if not os.path.isdir(os.path.join(REF, "powerba")):
        pytest.skip("baseline/_ref (the shipped reference package) is not installed")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import powerba.lm as ref_lm
    import paper_2204_12834_b200 as poba
    saved = {k: getattr(ref_lm, k) for k in ("blocks", "power_series_solve", "back_substitute",
                                             "residual_cost", "memory_account", "solvers")}
    # route 2: rebind the module globals lm.run resolves at call time
    ref_lm.blocks = types.SimpleNamespace(linearize=poba.linearize)
    ref_lm.power_series_solve = poba.power_series_solve
    ref_lm.back_substitute = poba.back_substitute
    ref_lm.residual_cost = poba.residual_cost
    ref_lm.memory_account = poba.memory_account
    ref_lm.solvers = poba.solvers
    yield ref_lm
    for k, v in saved.items():
        setattr(ref_lm, k, v)


def _ref_problem(name):
    from powerba.bal_io import BalProblem
    p, z = golden_problem(name)
    return BalProblem(p.camera_params, p.points, p.cam_indices, p.pt_indices, p.pixels, name=name), z


@pytest.mark.parametrize("name,tag,kw", [
    ("rig49", "lm_poba", dict(max_outer_iterations=50)),
    ("c2", "lm_c2", dict(max_outer_iterations=20, max_order=32, epsilon=1e-6)),
    ("c1", "lm_c1", dict(max_outer_iterations=10, max_order=32)),
])
def test_reference_lm_run_on_gpu_path(patched_ref, name, tag, kw):
    ref_lm = patched_ref
    bp, z = _ref_problem(name)
    tr = ref_lm.run(bp, ref_lm.LmConfig(**kw))
    costs = np.array([i.cost for i in tr.iterations])
    want = z[tag + "_cost"]
    assert len(costs) == len(want)
    assert np.all(np.abs(costs - want) <= COST_TOL * want)
    assert [i.accepted for i in tr.iterations] == z[tag + "_accepted"].tolist()
    assert [i.order_m for i in tr.iterations] == z[tag + "_order"].tolist()
    assert [i.lam for i in tr.iterations] == z[tag + "_lam"].tolist()
    assert [i.peak_bytes for i in tr.iterations] == z[tag + "_peak_bytes"].tolist()
    if name == "rig49":  # reference criterion 6 (pkg/test_output.txt:19)
        assert round(tr.final_cost, 4) == 7584.4992


def test_reference_evalkit_parallel_matches_sequential(patched_ref):
    """evalkit.run_benchmark(parallel=True) over the patched lm.run: the solver
    runs share one perturbed problem (one device context) from a thread pool."""
    from powerba import evalkit
    bp, _ = _ref_problem("c2")
    base = patched_ref.LmConfig(max_outer_iterations=8, max_order=20)
    specs = ["poba", "pcg", "poba32"]
    _, seq = evalkit.run_benchmark([("c2", bp)], specs, base, parallel=False)
    _, par = evalkit.run_benchmark([("c2", bp)], specs, base, parallel=True)
    for a, b in zip(seq, par):
        assert [i.cost for i in a.iterations] == [i.cost for i in b.iterations]
        assert [i.accepted for i in a.iterations] == [i.accepted for i in b.iterations]
