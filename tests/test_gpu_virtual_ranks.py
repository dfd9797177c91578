"""Sharded path on one B200: N virtual ranks in one process (poba_create_local).

The multi-GPU design partitions landmarks into
contiguous, observation-balanced ranges, keeps cameras replicated and ends
every series term with an all-reduce of the 9*n_cam camera vector.  With one
GPU per gpurun call, the ranks here are contexts on the same device driven by
one host thread each; their collectives meet at a host barrier (no kernel waits
on another rank) and reduce in rank order.  Everything else -- shard plan,
per-rank store and tiles, per-rank partial camera sums, replicated U^-1 / stop
test, local back-substitution, rank-ordered cost -- is the code the NCCL
contexts run.  The results must equal the single-context path (and, through
lm.run, the reference's own LM traces).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

from conftest import golden_problem

pytestmark = pytest.mark.gpu

COST_TOL = 1e-8   # north star: per-LM-iteration cost within 1e-8 relative
INC_TOL = 1e-9    # north star: increments within 1e-9 relative


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2204_12834_b200 as P
    return P


def _run_ranks(n, job):
    """Run job(rank, group) on n threads; returns the per-rank results in rank order."""
    from paper_2204_12834_b200 import _lib
    g = _lib.LocalGroup(n)
    out, errs = [None] * n, []

    def worker(r):
        try:
            out[r] = job(r, g)
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in th), "a virtual rank hung"
    if errs:
        raise errs[0][1]
    g.close()
    return out


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def _solve_all(dp, p, lam=1e-4):
    """The device calls of one LM iteration plus the PCG baseline, on one context."""
    from paper_2204_12834_b200 import _lib
    dev = dp.dev
    dev.set_points(p.points)
    bad = dev.linearize(p.camera_params)
    dev.damp(lam)
    x_forced, o_forced, _, _ = dev.series_solve(1e-300, 12)
    x, order, conv, ratios = dev.series_solve(0.01, 32, want_ratios=True)
    dl, nz = dev.back_substitute()
    cost0 = dev.cost(p.camera_params)
    cost1 = dev.cost(p.camera_params, trial=True)
    u0 = dev.read(_lib.READ_U0)
    bt = dev.read(_lib.READ_B_TILDE)
    sd = dev.schur_diagonal()
    xp, it, rel, pconv, _ = dev.pcg(_lib.PRECOND_SCHUR_JACOBI, 0, 1e-6, 60)
    info = dev.info()
    return dict(bad=bad, x_forced=x_forced, o_forced=o_forced, x=x, order=order, conv=conv, ratios=ratios,
                dl=dl, nz=nz, cost0=cost0, cost1=cost1, u0=u0, bt=bt, sd=sd, xp=xp, it=it, info=info)


def _problem(name):
    if name.startswith("cfg:"):
        from paper_2204_12834_b200 import configs
        cfg, scale = name[4:].split("@")
        return configs.make_config(cfg, float(scale), seed=0)
    return golden_problem(name)[0]


@pytest.mark.parametrize("name,n", [("c2", 2), ("mixed", 3), ("c2", 4), ("cfg:c3@0.1", 8), ("cfg:c4@0.01", 4)])
def test_virtual_ranks_match_single_context(P, name, n):
    from paper_2204_12834_b200 import blocks
    p = _problem(name)
    args = (p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)
    want = _solve_all(blocks.DeviceProblem(*args), p)

    def job(r, g):
        return _solve_all(blocks.DeviceProblem(*args, rank=r, nranks=n, group=g), p)

    got = _run_ranks(n, job)
    # the shard plan covers every landmark exactly once, in rank order
    assert got[0]["info"]["lm_lo"] == 0 and got[-1]["info"]["lm_hi"] == p.n_points
    for a, b in zip(got, got[1:]):
        assert a["info"]["lm_hi"] == b["info"]["lm_lo"]
    assert sum(g["info"]["n_obs_local"] for g in got) == len(p.cam_indices)
    for g in got:
        # the camera side is replicated: bitwise identical on every rank
        for key in ("x_forced", "x", "u0", "bt", "sd", "xp"):
            assert np.array_equal(g[key], got[0][key]), key
        assert (g["order"], g["conv"], g["it"], g["bad"]) == (got[0]["order"], got[0]["conv"], got[0]["it"],
                                                             got[0]["bad"])
        assert g["cost0"] == got[0]["cost0"] and g["cost1"] == got[0]["cost1"]
    r0 = got[0]
    assert r0["bad"] == want["bad"]
    assert _rel(r0["u0"], want["u0"]) <= 1e-13
    assert _rel(r0["bt"], want["bt"]) <= 1e-12
    assert _rel(r0["sd"], want["sd"]) <= 1e-12
    assert _rel(r0["x_forced"], want["x_forced"]) <= INC_TOL
    assert r0["order"] == want["order"] and r0["conv"] == want["conv"]
    assert _rel(r0["x"], want["x"]) <= INC_TOL
    assert abs(r0["it"] - want["it"]) <= 1
    assert _rel(r0["xp"], want["xp"]) <= 1e-5
    # back-substitution is local: each rank writes exactly its own landmarks
    dl = np.zeros_like(want["dl"])
    for g in got:
        lo, hi = g["info"]["lm_lo"], g["info"]["lm_hi"]
        own = np.zeros(p.n_points, bool)
        own[lo:hi] = True
        d = g["dl"].reshape(-1, 3)
        assert not np.any(d[~own]), "a rank wrote landmarks outside its shard"
        dl.reshape(-1, 3)[own] = d[own]
    assert _rel(dl, want["dl"]) <= INC_TOL
    for key in ("cost0", "cost1"):
        assert abs(r0[key][0] - want[key][0]) <= 1e-12 * want[key][0]
        assert r0[key][1] == want[key][1]


@pytest.mark.parametrize("name,tag,kw,n", [
    ("c1", "lm_c1", dict(max_outer_iterations=10, max_order=32), 2),
    ("c2", "lm_c2", dict(max_outer_iterations=20, max_order=32, epsilon=1e-6), 4),
    ("mixed", "lm_mixed", dict(max_outer_iterations=15, max_order=20), 3),
])
def test_virtual_ranks_lm_trace_matches_reference(P, name, tag, kw, n):
    """lm.run on every virtual rank reproduces the reference's own LM trace."""
    from paper_2204_12834_b200 import blocks
    p, z = golden_problem(name)
    args = (p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)

    def job(r, g):
        dp = blocks.DeviceProblem(*args, rank=r, nranks=n, group=g)
        return P.run(p, P.LmConfig(**kw), device_problem=dp)

    traces = _run_ranks(n, job)
    want = z[tag + "_cost"]
    for tr in traces:
        costs = np.array([i.cost for i in tr.iterations])
        assert len(costs) == len(want)
        assert np.all(np.abs(costs - want) <= COST_TOL * want)
        assert [i.accepted for i in tr.iterations] == z[tag + "_accepted"].tolist()
        assert [i.order_m for i in tr.iterations] == z[tag + "_order"].tolist()
        assert [i.lam for i in tr.iterations] == z[tag + "_lam"].tolist()
    assert all([i.cost for i in t.iterations] == [i.cost for i in traces[0].iterations] for t in traces)
