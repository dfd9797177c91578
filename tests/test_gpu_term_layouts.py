"""The term kernel's two camera-side layouts against the oracle and each other.

The store build picks `gather` (every tile gathers its 32 term records from L2;
1440 accumulator slots) or `table` (the chunk's term records in a second
shared-memory table, loaded per chunk at a round boundary; 896 slots) by a dry
run of the chunk cut (`poba_term_layout`; POBA_TERM_CHUNK_T forces one).  The
fixtures and C1-C4 take the table, C5 the gather, so both are forced here on
the same inputs: the mixed-track fixture (long landmarks, single-observation
points), C3 x 0.2 and C4 x 0.05 (several chunks per CTA range under the table
layout's smaller capacity).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

INC_TOL = 1e-9  # north star: increments within 1e-9 relative


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2204_12834_b200 as P
    return P


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def _problem(name):
    from paper_2204_12834_b200 import configs
    if name == "mixed":
        return configs.make_mixed_tracks()
    cfg, scale = name.split(":")
    return configs.make_config(cfg, float(scale), seed=0)


def _solve(P, p, layout, m, precision=64):
    """A fresh device store built under a forced layout: (info, W V^-1 W^T v, series x, back-substitution)."""
    from paper_2204_12834_b200 import _lib, blocks
    old = os.environ.get("POBA_TERM_CHUNK_T")
    os.environ["POBA_TERM_CHUNK_T"] = "1" if layout == "table" else "0"
    try:
        blocks.invalidate(p)
        s = P.assemble(p, lam=1e-4, precision=precision)
        s._activate()
        dev = s._dp.dev
        info = dev.info()
        v = np.random.default_rng(5).standard_normal(9 * p.n_cameras)
        wvw = dev.apply(_lib.OP_WVW, v)
        r = P.power_series_solve(s, 1e-300, m)
        dl = P.back_substitute(s, r.delta_p)
        return info, v, wvw, r, dl
    finally:
        if old is None:
            os.environ.pop("POBA_TERM_CHUNK_T", None)
        else:
            os.environ["POBA_TERM_CHUNK_T"] = old
        blocks.invalidate(p)


@pytest.mark.parametrize("name", ["mixed", "c3:0.2", "c4:0.05"])
def test_both_layouts_match_the_oracle(P, name):
    from oracle import poba_oracle as O
    p = _problem(name)
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    osys = O.OracleSystem(lin, 1e-4)
    m = 6
    x_want, _, _ = O.series_solve(osys, 1e-300, m)
    dl_want = O.back_sub(osys, x_want)
    got = {}
    for layout in ("gather", "table"):
        info, v, wvw, r, dl = _solve(P, p, layout, m)
        assert info["term_layout"] == layout
        want = osys.apply_w(osys.apply_v_inv(osys.apply_wt(v)))
        assert rel(wvw, want) <= 1e-12, layout
        assert r.order_used == m
        assert rel(r.delta_p, x_want) <= INC_TOL, layout
        assert rel(dl, dl_want) <= INC_TOL, layout
        got[layout] = (info, r.delta_p)
    # the table layout cuts chunks at rounds and has fewer slots: never fewer partials
    assert got["table"][0]["n_partials"] >= got["gather"][0]["n_partials"] or name == "mixed"
    assert rel(got["table"][1], got["gather"][1]) <= 1e-11


def test_layouts_are_bitwise_repeatable_and_poba32(P):
    p = _problem("c3:0.2")
    for layout in ("gather", "table"):
        a = _solve(P, p, layout, 4)
        b = _solve(P, p, layout, 4)
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3].delta_p, b[3].delta_p), layout
        assert np.array_equal(a[4], b[4]), layout
    x64 = _solve(P, p, "table", 4)[3].delta_p
    x32 = {layout: _solve(P, p, layout, 4, precision=32)[3].delta_p for layout in ("gather", "table")}
    assert rel(x32["table"], x32["gather"]) <= 1e-11   # same fp32-rounded blocks, different fixed summation order
    assert rel(x32["table"], x64) <= 1e-3               # fp32 storage, fp64 arithmetic


def test_automatic_choice(P):
    """The dry run takes the table when the camera working set fits (here: C3 x 0.2)."""
    from paper_2204_12834_b200 import blocks
    p = _problem("c3:0.2")
    os.environ.pop("POBA_TERM_CHUNK_T", None)
    blocks.invalidate(p)
    s = P.assemble(p, lam=1e-4)
    s._activate()
    assert s._dp.dev.info()["term_layout"] == "table"
    blocks.invalidate(p)


def test_sharded_virtual_ranks_in_both_layouts(P):
    """Two virtual ranks (the sharded path on one device) under each forced layout
    against the single context: same increments, each rank writes its own landmarks."""
    import threading

    from paper_2204_12834_b200 import _lib, blocks
    p = _problem("c3:0.1")
    ref = _solve(P, p, "table", 5)
    x_ref, dl_ref = ref[3].delta_p, ref[4]
    for layout in ("gather", "table"):
        os.environ["POBA_TERM_CHUNK_T"] = "1" if layout == "table" else "0"
        try:
            g = _lib.LocalGroup(2)
            out, errs = [None, None], []

            def worker(r):
                try:
                    dp = blocks.DeviceProblem(p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points,
                                              rank=r, nranks=2, group=g)
                    dev = dp.dev
                    assert dev.info()["term_layout"] == layout
                    dev.set_points(p.points)
                    dev.linearize(p.camera_params)
                    dev.damp(1e-4)
                    x, order, _, _ = dev.series_solve(1e-300, 5)
                    dl, _ = dev.back_substitute()
                    out[r] = (x, order, dl, dev.info())
                except BaseException as e:  # noqa: BLE001 - reported below
                    errs.append(e)

            th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
            for t in th:
                t.start()
            for t in th:
                t.join(timeout=600)
            assert not any(t.is_alive() for t in th), "a virtual rank hung"
            if errs:
                raise errs[0]
            g.close()
        finally:
            os.environ.pop("POBA_TERM_CHUNK_T", None)
        assert np.array_equal(out[0][0], out[1][0])  # camera side bitwise identical on both ranks
        assert out[0][1] == out[1][1] == 5
        assert rel(out[0][0], x_ref) <= INC_TOL, layout
        dl = np.zeros_like(dl_ref)
        for r in range(2):
            lo, hi = out[r][3]["lm_lo"], out[r][3]["lm_hi"]
            dl.reshape(-1, 3)[lo:hi] = out[r][2].reshape(-1, 3)[lo:hi]
        assert rel(dl, dl_ref) <= INC_TOL, layout
