"""Pipelined landmark transfers (``-m gpu``): the points upload overlapped with
the Jacobian pass and the Delta x_l download overlapped with back-substitution
must give bitwise the same results as the plain transfers, for pageable and
page-locked host arrays, with long landmarks present (``mixed``) and without.
``POBA_XFER_MIN_BYTES`` forces the pipelined path at test sizes.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(name):
    from paper_2204_12834_b200 import configs
    return configs.make_mixed_tracks() if name == "mixed" else configs.make_config(name, 0.1)


def _run(dev, p, cams, pts, pinned_out):
    from paper_2204_12834_b200 import _lib
    dev.linearize(cams, pts)
    dev.damp(1e-4)
    reads = [dev.read(k).copy() for k in (_lib.READ_U0, _lib.READ_V0, _lib.READ_B_P, _lib.READ_B_L,
                                           _lib.READ_D_P, _lib.READ_D_L)]
    dev.series_solve(1e-2, 20)
    if pinned_out:
        import torch
        dl = torch.zeros(3 * p.n_points, dtype=torch.float64, pin_memory=True).numpy()
    else:
        dl = np.zeros(3 * p.n_points)
    _lib._check(dev._lib.poba_back_substitute(dev._h, None, _lib._d(dl), None))
    return reads, dl.copy(), dev.get_points().copy()


@pytest.mark.parametrize("name", ["mixed", "c3"])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipelined_transfers_match_plain(name, pinned, monkeypatch):
    import torch
    import paper_2204_12834_b200 as P
    p = _problem(name)
    s = P.assemble(p, lam=1e-4)
    s._activate()
    dev = s._dp.dev
    cams, pts = p.camera_params, np.array(p.points)
    pts = pts + 1e-3 * np.random.default_rng(0).standard_normal(pts.shape)  # not the points already on the device
    if pinned:
        pts = torch.from_numpy(pts).pin_memory().numpy()
    monkeypatch.setenv("POBA_XFER_MIN_BYTES", str(1 << 62))
    plain = _run(dev, p, cams, pts, pinned)
    monkeypatch.setenv("POBA_XFER_MIN_BYTES", "0")
    piped = _run(dev, p, cams, pts, pinned)
    for a, b in zip(plain[0], piped[0]):
        assert np.array_equal(a, b)
    assert np.array_equal(plain[1], piped[1])
    assert np.array_equal(plain[2], piped[2])
    assert np.array_equal(piped[2], np.asarray(pts))
