"""Problem container with the reference's array layout (the drop-in input contract).

Mirrors ``powerba.bal_io.BalProblem`` (reference ``pkg/src/powerba/bal_io.py:55-129``):
``camera_params`` (n_cameras, 9) float64 in BAL order [rotvec, t, f, k1, k2],
``points`` (n_points, 3) float64, ``cam_indices``/``pt_indices`` int64 (n_obs,),
``pixels`` (n_obs, 2) float64, all C-contiguous.  Every entry point of this package
also accepts the reference's own ``BalProblem`` (duck typing on these attributes).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

CAMERA_PARAMS = 9
POINT_PARAMS = 3


@dataclass
class Problem:
    camera_params: np.ndarray
    points: np.ndarray
    cam_indices: np.ndarray
    pt_indices: np.ndarray
    pixels: np.ndarray
    name: str = ""
    n_pruned_cameras: int = 0
    n_pruned_points: int = 0

    def __post_init__(self) -> None:
        # same validation, same messages as bal_io.py:79-98
        self.camera_params = np.ascontiguousarray(self.camera_params, dtype=np.float64)
        self.points = np.ascontiguousarray(self.points, dtype=np.float64)
        self.cam_indices = np.ascontiguousarray(self.cam_indices, dtype=np.int64)
        self.pt_indices = np.ascontiguousarray(self.pt_indices, dtype=np.int64)
        self.pixels = np.ascontiguousarray(self.pixels, dtype=np.float64)
        if self.camera_params.ndim != 2 or self.camera_params.shape[1] != CAMERA_PARAMS:
            raise ValueError("camera_params must have shape (n_cameras, 9)")
        if self.points.ndim != 2 or self.points.shape[1] != POINT_PARAMS:
            raise ValueError("points must have shape (n_points, 3)")
        n_obs = self.cam_indices.shape[0]
        if self.pt_indices.shape != (n_obs,) or self.pixels.shape != (n_obs, 2):
            raise ValueError("observation arrays have inconsistent lengths")
        if n_obs == 0:
            raise ValueError("problem has no observations")
        if self.cam_indices.min() < 0 or self.cam_indices.max() >= self.n_cameras:
            raise ValueError("camera index out of range")
        if self.pt_indices.min() < 0 or self.pt_indices.max() >= self.n_points:
            raise ValueError("point index out of range")
        key = self.cam_indices * self.n_points + self.pt_indices
        if not (key[1:] > key[:-1]).all():  # sorted input (BAL order) needs no sort
            if np.unique(key).size != n_obs:
                raise ValueError("duplicate (camera, point) observation")
        if np.bincount(self.cam_indices, minlength=self.n_cameras).min() == 0:
            raise ValueError("every camera must have at least one observation")
        if np.bincount(self.pt_indices, minlength=self.n_points).min() == 0:
            raise ValueError("every point must have at least one observation")

    @property
    def n_cameras(self) -> int:
        return self.camera_params.shape[0]

    @property
    def n_points(self) -> int:
        return self.points.shape[0]

    @property
    def n_observations(self) -> int:
        return self.cam_indices.shape[0]

    def copy(self) -> "Problem":
        return replace(self, camera_params=self.camera_params.copy(), points=self.points.copy(),
                       cam_indices=self.cam_indices.copy(), pt_indices=self.pt_indices.copy(),
                       pixels=self.pixels.copy())

    def fingerprint(self) -> str:
        """sha256 over the five arrays, used to tie fixtures to generated inputs."""
        import hashlib
        h = hashlib.sha256()
        for a in (self.camera_params, self.points, self.cam_indices, self.pt_indices, self.pixels):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()
