"""Multi-GPU protocol on CPU: 2 gloo ranks, landmark shards from libpoba's own planner.

The sharded GPU path partitions landmarks into contiguous ranges
(`poba_shard_bounds`, the same plan `poba_create_sharded` contexts use), keeps
cameras replicated, all-reduces the 9*n_cam camera vector once per series term
and once per linearization (U0, b_p), and evaluates U^-1, the partial sum and
the stop test replicated.  Here every rank runs that protocol with the CPU
oracle's arithmetic on its shard and torch.distributed (gloo) as the exchange;
the result must equal the unsharded oracle.  No kernel is launched.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import REPO, golden_problem


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_solve(rank, world, port, out):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import poba_oracle as O
    from paper_2204_12834_b200 import _lib
    from conftest import golden_problem as gp

    p, _ = gp("c1")
    lam, eps, m = 1e-4, 1e-300, 12
    k = np.bincount(p.pt_indices, minlength=p.n_points)
    bounds = _lib.shard_bounds(k, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    sel = np.flatnonzero((p.pt_indices >= lo) & (p.pt_indices < hi))
    ci, pi = p.cam_indices[sel], p.pt_indices[sel]
    _, jp, jl, _ = O.project(p.camera_params[ci], p.points[pi], p.pixels[sel], True)
    res, _ = O.project(p.camera_params[ci], p.points[pi], p.pixels[sel], False)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    n_c = p.n_cameras
    # linearization: camera side all-reduced, landmark side local
    U0 = np.zeros((n_c, 9, 9))
    bp = np.zeros((n_c, 9))
    np.add.at(U0, ci, np.einsum("oai,oaj->oij", jp, jp))
    np.add.at(bp, ci, np.einsum("oai,oa->oi", jp, res))
    U0, bp = allreduce(U0), allreduce(bp).ravel()
    V0 = np.zeros((p.n_points, 3, 3))
    bl = np.zeros((p.n_points, 3))
    np.add.at(V0, pi, np.einsum("oai,oaj->oij", jl, jl))
    np.add.at(bl, pi, np.einsum("oai,oa->oi", jl, res))
    ii = np.arange(9)
    Dp = np.sqrt(np.clip(U0[:, ii, ii], 1e-12, 1e12))
    U = U0.copy()
    U[:, ii, ii] += lam * Dp ** 2
    Ui = O.spd_inverse(U, "damped pose")
    mine = np.arange(lo, hi)
    ii = np.arange(3)
    Dl = np.sqrt(np.clip(V0[mine][:, ii, ii], 1e-12, 1e12))
    V = V0[mine].copy()
    V[:, ii, ii] += lam * Dl ** 2
    Vi = np.zeros((p.n_points, 3, 3))
    Vi[mine] = O.spd_inverse(V, "damped point")

    def w_local(z_pts):  # camera vector of this shard's observations
        g = np.einsum("oab,ob->oa", jl, z_pts[pi])
        out = np.zeros((n_c, 9))
        np.add.at(out, ci, np.einsum("oai,oa->oi", jp, g))
        return out

    def wt_local(t):
        u = np.einsum("oai,oi->oa", jp, t.reshape(n_c, 9)[ci])
        y = np.zeros((p.n_points, 3))
        np.add.at(y, pi, np.einsum("oab,oa->ob", jl, u))
        return y

    z = np.einsum("pij,pj->pi", Vi, bl)
    bt = bp - allreduce(w_local(z)).ravel()                     # one all-reduce per damp
    t = np.einsum("pij,pj->pi", Ui, -bt.reshape(n_c, 9)).ravel()
    x = t.copy()
    for _ in range(m):                                           # one all-reduce per term
        y = wt_local(t)
        z = np.einsum("pij,pj->pi", Vi, y)
        r = allreduce(w_local(z))
        t = np.einsum("pij,pj->pi", Ui, r).ravel()
        x = x + t
    dl = -np.einsum("pij,pj->pi", Vi, bl + wt_local(x))[mine]   # back-substitution stays local
    out.put((rank, lo, hi, x, dl, U0, bp))
    dist.destroy_process_group()


def test_two_rank_landmark_sharding_matches_unsharded():
    import torch.multiprocessing as mp
    from oracle import poba_oracle as O
    p, _ = golden_problem("c1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_solve, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    s = O.OracleSystem(lin, 1e-4)
    want, _, _ = O.series_solve(s, 1e-300, 12)
    want_l = O.back_sub(s, want).reshape(-1, 3)
    (_, lo0, hi0, x0, dl0, U00, bp0), (_, lo1, hi1, x1, dl1, _, _) = outs
    assert lo0 == 0 and hi0 == lo1 and hi1 == p.n_points
    assert np.array_equal(x0, x1)  # replicated camera side: bit-identical on every rank
    assert np.linalg.norm(x0 - want) <= 1e-12 * np.linalg.norm(want)
    assert np.linalg.norm(U00 - lin.U0) <= 1e-13 * np.linalg.norm(lin.U0)
    got_l = np.concatenate([dl0, dl1])
    assert np.linalg.norm(got_l - want_l) <= 1e-12 * np.linalg.norm(want_l)


def test_shard_bounds_are_landmark_complete_and_balanced():
    from paper_2204_12834_b200 import _lib, configs
    p = configs.make_config("c4", 0.01)
    k = np.bincount(p.pt_indices, minlength=p.n_points)
    for n in (1, 2, 4, 8):
        b = _lib.shard_bounds(k, n)
        assert b[0] == 0 and b[-1] == p.n_points and np.all(np.diff(b) > 0)
        obs = np.array([k[b[r]:b[r + 1]].sum() for r in range(n)])
        assert obs.max() <= obs.mean() * 1.05 + 64
    with pytest.raises(ValueError, match="observed"):
        _lib.shard_bounds(np.array([1, 0, 2]), 2)
