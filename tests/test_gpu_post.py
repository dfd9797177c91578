"""GPU PoST (clustered solve on a virtual-landmark store, per-cluster stop tests) vs the reference.

Golden: tests/golden/post.npz from the reference's clustering.cluster_cameras,
solve_clustered and lm.run(solver="post") (tests/golden/make_golden.py).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_problem, load_golden

pytestmark = pytest.mark.gpu

POST = {"c1": "c1", "mixed": "mixed"}


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d else 1.0)


@pytest.mark.parametrize("tag", sorted(POST))
def test_clustered_solve(tag):
    import paper_2204_12834_b200 as P
    from paper_2204_12834_b200 import clustering
    p, _ = golden_problem(POST[tag])
    z = load_golden("post")
    lin = P.linearize(p)
    for size in (1, 5, 16, 1000):
        pre = f"{tag}_s{size}_"
        part = clustering.cluster_cameras(p, size)
        assert np.array_equal(part.assignment, z[pre + "assignment"])
        assert [part.n_clusters, part.cut_observations] == z[pre + "meta"].tolist()
        for j, lam in enumerate([1e-4, 1.0]):
            s = lin.damp(lam)
            for k, (eps, m) in enumerate([(0.01, 20), (1e-300, 6)]):
                q = pre + f"l{j}_e{k}_"
                r = clustering.solve_clustered(s, part, eps, m)
                assert [r.order_used, r.converged] == z[q + "order_conv"].tolist(), (size, lam, eps)
                # singleton clusters split every landmark into k = 1 virtual landmarks whose damped
                # V (rank-2 V0 + lam D^2) has condition ~1/lam: the fp64 noise floor is ~1e-9 there
                tol = 1e-8 if size == 1 else 1e-9
                assert rel(r.delta_p, z[q + "delta_p"]) < tol, (size, lam, eps, rel(r.delta_p, z[q + "delta_p"]))


def test_single_cluster_equals_plain_series():
    """One cluster holding every camera is the unclustered solve (clustering.py:110-112)."""
    import paper_2204_12834_b200 as P
    from paper_2204_12834_b200 import clustering
    p, _ = golden_problem("c1")
    s = P.assemble(p, lam=1e-4)
    part = clustering.cluster_cameras(p, 10_000)
    assert part.n_clusters == 1
    r = clustering.solve_clustered(s, part, 0.01, 20)
    q = P.power_series_solve(s, 0.01, 20)
    assert r.order_used == q.order_used and r.converged == q.converged
    assert rel(r.delta_p, q.delta_p) < 1e-12


def test_restrict_system_matches_virtual_store():
    import paper_2204_12834_b200 as P
    from paper_2204_12834_b200 import clustering
    p, _ = golden_problem("mixed")
    s = P.assemble(p, lam=1e-2)
    part = clustering.cluster_cameras(p, 16)
    r = clustering.solve_clustered(s, part, 1e-300, 5)
    for c in range(part.n_clusters):
        cams = np.flatnonzero(part.assignment == c)
        sub = clustering.restrict_system(s, cams)
        q = P.power_series_solve(sub, 1e-300, 5)
        assert rel(q.delta_p, r.delta_p.reshape(-1, 9)[cams].ravel()) < 1e-10


@pytest.mark.parametrize("tag", sorted(POST))
def test_lm_post_trace(tag):
    import paper_2204_12834_b200 as P
    p, _ = golden_problem(POST[tag])
    z = load_golden("post")
    t = f"{tag}_lm_post"
    tr = P.run(p, P.LmConfig(solver="post", max_cluster_size=5, max_outer_iterations=10, max_order=20))
    costs = np.array([i.cost for i in tr.iterations])
    want = z[t + "_cost"]
    assert len(costs) == len(want)
    assert np.all(np.abs(costs - want) <= 1e-8 * want)
    assert [i.accepted for i in tr.iterations] == z[t + "_accepted"].tolist()
    assert [i.order_m for i in tr.iterations][1:] == z[t + "_order"].tolist()[1:]
