"""Dense direct baseline (device Schur columns, host Cholesky) vs the reference's dense_direct."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_problem, load_golden

pytestmark = pytest.mark.gpu
PROBLEMS = {"c1": "c1", "noisy": "noisy4x60"}


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
def test_dense_direct_and_lm(tag):
    import paper_2204_12834_b200 as P
    from paper_2204_12834_b200 import solvers
    p, _ = golden_problem(PROBLEMS[tag])
    z = load_golden("direct")
    lin = P.linearize(p)
    # the dense solve inherits kappa(S) (~1e8 at lambda = 1e-4) on fp64 rounding of S's columns
    for j, (lam, tol) in enumerate([(1e-4, 1e-6), (1.0, 1e-10)]):
        assert rel(solvers.dense_direct(lin.damp(lam)), z[f"{tag}_l{j}_delta_p"]) < tol
    tr = P.run(p, P.LmConfig(solver="direct", max_outer_iterations=10))
    want = z[f"{tag}_lm_direct_cost"]
    costs = np.array([i.cost for i in tr.iterations])
    assert len(costs) == len(want) and np.all(np.abs(costs - want) <= 1e-8 * want)
    assert [i.accepted for i in tr.iterations] == z[f"{tag}_lm_direct_accepted"].tolist()


def test_dense_direct_refuses_large():
    import paper_2204_12834_b200 as P
    from paper_2204_12834_b200 import configs, solvers
    p = configs.make_config("c3", 0.25)  # 300 cameras -> 2700 pose parameters
    assert 9 * p.n_cameras > solvers.DENSE_DIM_LIMIT
    with pytest.raises(ValueError, match="dense solve refused"):
        solvers.dense_direct(P.assemble(p, lam=1e-4))
