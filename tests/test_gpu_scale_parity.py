"""Parity against the oracle at configuration scale (about a million observations).

The golden fixtures pin the path on small problems; these cases run the fused
term kernel on full-size store layouts -- hundreds of chunks per CTA range,
bank-coloured accumulator slots, tiles whose distinct cameras collide in the
shared-memory banks, long landmarks (C4's heavy-tailed tracks) -- and compare
with the oracle (the reference algorithm restated in numpy) on the same inputs:
one W V^-1 W^T pass, a forced power series and the back-substitution.
"""
from __future__ import annotations

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


@pytest.mark.parametrize("name,scale", [("c3", 1.0), ("c4", 0.1)])
def test_operators_and_series_at_scale(P, name, scale):
    from oracle import poba_oracle as O
    from paper_2204_12834_b200 import _lib, configs
    p = configs.make_config(name, scale, seed=0)
    lam = 1e-4
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    osys = O.OracleSystem(lin, lam)
    s = P.assemble(p, lam=lam)
    s._activate()
    dev = s._dp.dev
    v = np.random.default_rng(11).standard_normal(9 * p.n_cameras)
    want = osys.apply_w(osys.apply_v_inv(osys.apply_wt(v)))
    got = dev.apply(_lib.OP_WVW, v)
    assert rel(got, want) <= 1e-12
    m = 6
    x_want, _, _ = O.series_solve(osys, 1e-300, m)
    r = P.power_series_solve(s, 1e-300, m)
    assert r.order_used == m
    assert rel(r.delta_p, x_want) <= INC_TOL
    dl_want = O.back_sub(osys, x_want)
    dl = P.back_substitute(s, r.delta_p)
    assert rel(dl, dl_want) <= INC_TOL
