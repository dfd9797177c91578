"""Camera-model helpers that stay on the host.

The residual and Jacobian of the 9-parameter BAL camera (reference
``pkg/src/powerba/camera.py:67-135``) are evaluated by libpoba kernels.  The
rotation retraction of the LM state update touches only 9 n_cameras values and
stays on the host exactly as the reference does it (``camera.py:160-166``,
scipy quaternion composition), so accepted states match the reference bit for
bit given the same increments.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial.transform import Rotation

MIN_PROJECTED_DEPTH = 1e-12  # camera.py:22, enforced in the device kernels
POSE_DIM = 9
POINT_DIM = 3


def rotation_matrices(rotvecs: np.ndarray) -> np.ndarray:
    """Axis-angle vectors (n, 3) to rotation matrices (n, 3, 3) (camera.py:49-51)."""
    return Rotation.from_rotvec(np.atleast_2d(rotvecs)).as_matrix()


def compose_rotations(rotvecs: np.ndarray, deltas: np.ndarray) -> np.ndarray:
    """Right-multiply increments onto rotation vectors: log(R(w) Exp(delta)) (camera.py:160-166)."""
    r = Rotation.from_rotvec(np.atleast_2d(rotvecs)) * Rotation.from_rotvec(np.atleast_2d(deltas))
    return r.as_rotvec()
