"""Host logic of the device-store cache (blocks.device_problem): what a cached
store is validated against, and that large problems' arrays are locked against
in-place edits until ``invalidate``.  No GPU needed (no context is created)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2204_12834_b200 import blocks
from paper_2204_12834_b200.problem import Problem


def _problem(n_obs):
    rng = np.random.default_rng(0)
    cams = rng.standard_normal((4, 9))
    pts = rng.standard_normal((n_obs // 4, 3))
    ci = np.arange(n_obs) % 4                 # every (camera, point) pair once
    pi = np.arange(n_obs) // 4
    return Problem(cams, pts, ci, pi, rng.standard_normal((n_obs, 2)), name="t")


def test_small_problem_snapshot_is_a_full_copy():
    p = _problem(64)
    snap = blocks._snapshot(p)
    assert snap[0] == "copy" and blocks._same_snapshot(p, snap)
    p.pixels[3, 1] += 1.0
    assert not blocks._same_snapshot(p, snap)
    assert p.pixels.flags.writeable


def test_large_problem_arrays_locked_until_invalidate(monkeypatch):
    monkeypatch.setattr(blocks, "_FULL_COPY_OBS", 16)
    p = _problem(64)
    snap = blocks._snapshot(p)
    assert snap[0] == "locked" and blocks._same_snapshot(p, snap)
    with pytest.raises(ValueError):
        p.pixels[0, 0] = 1.0
    with pytest.raises(ValueError):
        p.cam_indices[0] = 1
    object.__setattr__(p, "_poba_device", (blocks._signature(p), snap, None))
    blocks.invalidate(p)
    assert not hasattr(p, "_poba_device")
    p.pixels[0, 0] = 1.0  # writable again


def test_large_problem_views_use_a_digest(monkeypatch):
    monkeypatch.setattr(blocks, "_FULL_COPY_OBS", 16)
    p = _problem(64)
    base = np.zeros((128, 2))
    base[:64] = p.pixels
    object.__setattr__(p, "pixels", base[:64])  # a view: cannot be locked
    snap = blocks._snapshot(p)
    assert snap[0] == "digest" and blocks._same_snapshot(p, snap)
    base[5, 0] += 1.0
    assert not blocks._same_snapshot(p, snap)


def test_frozen_state_copies_small_and_fingerprints_large(monkeypatch):
    cams, pts = np.ones((2, 9)), np.ones((10, 3))
    c2, p2, fp = blocks._frozen_state(cams, pts)
    assert fp is None and p2 is not pts and c2 is not cams
    monkeypatch.setattr(blocks, "_STATE_COPY_BYTES", 8)
    c2, p2, fp = blocks._frozen_state(cams, pts)
    assert p2 is pts and np.array_equal(pts[fp[0]], fp[1])
