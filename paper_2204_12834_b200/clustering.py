"""PoST: covisibility clustering of cameras and per-cluster pose solves, on the GPU.

Drop-in for the reference module ``powerba.clustering`` (reference
``pkg/src/powerba/clustering.py:24-148``).  ``cluster_cameras`` runs the
reference's greedy heaviest-edge merge in libpoba's host C++
(``poba_cluster_cameras``).  ``solve_clustered`` does not build one
sub-problem per cluster: it keeps a second device store in which every
(landmark, cluster) pair is its own virtual landmark, so the reduced system is
block diagonal over the clusters and each fused series-term pass advances all
clusters at once, with a separate stop test per cluster
(``poba_series_solve_clustered``).  The virtual landmarks keep the global
landmark damping diagonal, as ``restrict_system`` keeps it.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .blocks import POSE_DIM, DeviceProblem, assemble_from_observations
from .power_series import _device_system

__all__ = ["CameraClustering", "ClusteredSolveResult", "cluster_cameras", "restrict_system", "solve_clustered"]


@dataclass(frozen=True)
class CameraClustering:
    """Partition of the cameras plus cut statistics (clustering.py:24-37)."""

    assignment: np.ndarray  # (n_cameras,) cluster id per camera
    n_clusters: int
    sizes: np.ndarray
    cut_observations: int


@dataclass(frozen=True)
class ClusteredSolveResult:
    delta_p: np.ndarray
    order_used: int      # max over clusters
    converged: bool      # all clusters met the stop criterion


def cluster_cameras(problem, max_cluster_size: int, seed: int = 0) -> CameraClustering:
    """Greedy agglomerative merge along covisibility edges, heaviest first (clustering.py:49-101)."""
    del seed  # tie-break is by index, as in the reference
    if max_cluster_size < 1:
        raise ValueError("max_cluster_size must be at least 1")
    assignment, n_clusters, cut = _lib.cluster_cameras(problem.n_cameras, problem.n_points, problem.cam_indices,
                                                       problem.pt_indices, max_cluster_size)
    return CameraClustering(assignment, n_clusters, np.bincount(assignment, minlength=n_clusters), cut)


def restrict_system(system, cluster_cams: np.ndarray):
    """The sub-system of one camera cluster (clustering.py:104-122), as its own device system."""
    sys_ = _device_system(system)
    store = sys_.store
    cluster_cams = np.asarray(cluster_cams, dtype=np.int64)
    cam_in = np.zeros(store.n_cameras, dtype=bool)
    cam_in[cluster_cams] = True
    cam_map = np.full(store.n_cameras, -1, dtype=np.int64)
    cam_map[cluster_cams] = np.arange(len(cluster_cams))
    mask = cam_in[store.cam_sorted]
    pt_kept = store.pt_sorted[mask]
    kept_lms = np.unique(pt_kept)
    lm_map = np.full(store.n_points, -1, dtype=np.int64)
    lm_map[kept_lms] = np.arange(len(kept_lms))
    rows = store.storage_obs[mask]
    lin = assemble_from_observations(cam_map[store.cam_sorted[mask]], lm_map[pt_kept], rows[:, :, 0:POSE_DIM],
                                     rows[:, :, POSE_DIM:POSE_DIM + 3], rows[:, :, -1],
                                     n_cameras=len(cluster_cams), n_points=len(kept_lms),
                                     precision=sys_.lin.precision)
    lin._dp.dev.set_dl(sys_.lin.D_l[kept_lms])
    lin._cache["D_l"] = sys_.lin.D_l[kept_lms]
    return lin.damp(sys_.lam, sys_.damping)


class _VirtualStore:
    """Second device store: one virtual landmark per (landmark, cluster) pair."""

    def __init__(self, dp: DeviceProblem, assignment: np.ndarray, n_clusters: int):
        cl = assignment[np.asarray(dp.cam_indices)]
        key = np.asarray(dp.pt_indices, dtype=np.int64) * n_clusters + cl
        uniq, virt = np.unique(key, return_inverse=True)
        self.to_point = uniq // n_clusters
        self.assignment, self.n_clusters = assignment, n_clusters
        self.dp = DeviceProblem(dp.cam_indices, virt.astype(np.int64), dp.pixels, dp.n_cameras, len(uniq),
                                device=dp.dev.device)

    def linearize_like(self, lin):
        """Linearize the virtual store at the same source (state or explicit rows) as ``lin``."""
        dev = self.dp.dev
        dev.set_precision(lin.precision)
        src = lin._source
        if src[0] == "state":
            dev.linearize(src[1], np.asarray(src[2])[self.to_point])
        else:
            dev.linearize_explicit(*src[1:])
        dev.set_dl(np.asarray(lin.D_l)[self.to_point])


def _virtual_store(sys_, partition: CameraClustering) -> _VirtualStore:
    dp = sys_._dp
    key = (partition.n_clusters, partition.assignment.tobytes())
    cached = getattr(dp, "_post_store", None)
    if cached is None or cached[0] != key:
        cached = (key, _VirtualStore(dp, np.asarray(partition.assignment), partition.n_clusters))
        dp._post_store = cached
    return cached[1]


def solve_clustered(system, partition: CameraClustering, epsilon: float = 0.01,
                    max_order: int = 20) -> ClusteredSolveResult:
    """Per-cluster truncated-series pose steps, concatenated globally (clustering.py:125-148)."""
    sys_ = _device_system(system)
    if partition.assignment.shape[0] != sys_.n_cameras:
        raise ValueError("partition does not match the system's camera count")
    with sys_._dp.lock:
        vs = _virtual_store(sys_, partition)
        vs.linearize_like(sys_.lin)
        vs.dp.dev.damp(sys_.lam, sys_.damping == "identity")
        dp, order, conv = vs.dp.dev.series_solve_clustered(partition.assignment, partition.n_clusters, epsilon,
                                                           max_order)
    return ClusteredSolveResult(dp, order, conv)
