"""Shared pytest configuration: the ``gpu`` marker and golden-fixture loaders."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def golden_problem(name):
    """Rebuild the fixture's problem (inputs stored, or regenerated and fingerprint-checked)."""
    from paper_2204_12834_b200.problem import Problem
    z = load_golden(name)
    if "camera_params" in z:
        p = Problem(z["camera_params"], z["points"], z["cam_indices"], z["pt_indices"], z["pixels"],
                    name=name)
    else:
        from paper_2204_12834_b200 import configs
        p = configs.make_config(name)
    assert p.fingerprint() == str(z["fingerprint"]), f"{name}: regenerated inputs drifted"
    return p, z


@pytest.fixture(scope="session")
def golden():
    return load_golden
