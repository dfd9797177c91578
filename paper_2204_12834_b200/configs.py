"""Seeded synthetic bundle-adjustment problems for the five BASELINE.json configs.

The paper evaluates on the BAL dataset, which is not available here; these
generators stand in for it with the shapes, track-length distributions and
noise models that BASELINE.json names.  They are host code (numpy) and emit
arrays in the reference's ``BalProblem`` layout (reference
``pkg/src/powerba/bal_io.py:55-98``), satisfying its validation: every camera
and point observed, unique (camera, point) pairs, points in front of the
camera (negative camera-frame z, reference ``synthetic.py:17-31``).

Interpretation choices (recorded in DESIGN.md):
  * "k1/k2 ~ N(0, 1e-3)" is read as standard deviation 1e-3.
  * "0.01 rad rotation / 0.05 translation": each camera is turned by a
    right-multiplied random rotation (per-axis standard deviation 0.01) about its
    own centre, and its centre moved by N(0, 0.05^2 I) (the reference ``perturb``
    never touches rotations, ``bal_io.py:297-312``; the configs ask for it).
  * Landmark indices are emitted in a spatially coherent order (sorted along
    the scene), and observations in BAL file order (camera, then point).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.spatial.transform import Rotation

from .problem import Problem

# generator-side depth margin: every observed point is at least this far in front of
# its camera, so the 0.01 rad / 0.05 perturbation cannot push it near the image plane
MIN_DEPTH = 1.0


@dataclass(frozen=True)
class LmSettings:
    max_outer_iterations: int = 50
    max_order: int = 20
    epsilon: float = 0.01
    initial_lambda: float = 1e-4


# BASELINE.json configs[0..4]; LM/series settings as the configs state them
LM_SETTINGS = {
    "c1": LmSettings(max_outer_iterations=10, max_order=32, epsilon=0.01),
    "c2": LmSettings(max_outer_iterations=20, max_order=32, epsilon=1e-6),
    "c3": LmSettings(max_outer_iterations=50, max_order=32, epsilon=0.01),
    "c3m64": LmSettings(max_outer_iterations=50, max_order=64, epsilon=0.01),
    "c4": LmSettings(),
    "c5": LmSettings(max_outer_iterations=50, max_order=32, epsilon=0.01),
}


# ---------------------------------------------------------------------------
# geometry helpers
# ---------------------------------------------------------------------------

def _frames(centers, forward, up_hint=(0.0, 0.0, 1.0)):
    """World->camera rotations whose camera z axis is -forward (points in front: z<0)."""
    f = forward / np.linalg.norm(forward, axis=1, keepdims=True)
    z = -f
    up = np.broadcast_to(np.asarray(up_hint, dtype=np.float64), z.shape).copy()
    near = np.abs(np.einsum("ij,ij->i", up, z)) > 0.95
    up[near] = (1.0, 0.0, 0.0)
    x = np.cross(up, z)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = np.cross(z, x)
    R = np.stack([x, y, z], axis=1)
    return R


def _cameras(centers, R, rng, focal=500.0, dist_sigma=1e-3):
    n = len(centers)
    cams = np.empty((n, 9))
    cams[:, 0:3] = Rotation.from_matrix(R).as_rotvec()
    Rm = Rotation.from_rotvec(cams[:, 0:3]).as_matrix()
    cams[:, 3:6] = -np.einsum("nij,nj->ni", Rm, centers)
    cams[:, 6] = focal
    cams[:, 7] = rng.normal(0.0, dist_sigma, n)
    cams[:, 8] = rng.normal(0.0, dist_sigma, n)
    return cams


def _camera_frame(cams, cam_ids, X, batch=1 << 21):
    """Camera-frame points P = R(w) X + t for parallel (cam_ids, X)."""
    Rc = Rotation.from_rotvec(cams[:, 0:3]).as_matrix()
    out = np.empty((len(cam_ids), 3))
    for a in range(0, len(cam_ids), batch):
        c = cam_ids[a:a + batch]
        out[a:a + batch] = np.einsum("nij,nj->ni", Rc[c], X[a:a + batch]) + cams[c, 3:6]
    return out


def _pixels(cams, cam_ids, X, P=None):
    P = _camera_frame(cams, cam_ids, X) if P is None else P
    p = -P[:, 0:2] / P[:, 2:3]
    s = np.einsum("ni,ni->n", p, p)
    c = cams[cam_ids]
    d = 1.0 + s * (c[:, 7] + c[:, 8] * s)
    return (c[:, 6] * d)[:, None] * p


def _visible(P, tan_h=1.0, tan_v=1.0):
    z = P[..., 2]
    front = z < -MIN_DEPTH
    zs = np.where(front, z, -1.0)
    return front & (np.abs(P[..., 0] / zs) < tan_h) & (np.abs(P[..., 1] / zs) < tan_v)


def _morton2(ix, iy):
    def spread(v):
        v = v.astype(np.uint64) & np.uint64(0xFFFF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v
    return spread(ix) | (spread(iy) << np.uint64(1))


def _pick(cands, valid, k):
    """Per row take the first k valid, distinct entries of ``cands`` (already random order).

    Returns (row, value, n_distinct_valid) arrays.
    """
    n, m = cands.shape
    key = np.where(valid, cands, -1 - np.arange(m)[None, :])
    srt = np.argsort(key, axis=1, kind="stable")
    sk = np.take_along_axis(key, srt, axis=1)
    first_s = np.ones((n, m), dtype=bool)
    first_s[:, 1:] = sk[:, 1:] != sk[:, :-1]
    first = np.empty_like(first_s)
    np.put_along_axis(first, srt, first_s, axis=1)
    ok = valid & first
    rank = np.cumsum(ok, axis=1) - 1
    take = ok & (rank < np.asarray(k)[:, None])
    rows, cols = np.nonzero(take)
    return rows, cands[rows, cols], ok.sum(axis=1)


def _finish(name, cams_true, X_true, cam_idx, pt_idx, rng, *, outlier_frac=0.0,
            outlier_px=50.0, pixel_sigma=1.0, rot_sigma=0.01, t_sigma=0.05, pt_sigma=0.05):
    """Sort to BAL file order, synthesize noisy pixels, perturb the initial state."""
    o = np.lexsort((pt_idx, cam_idx))
    cam_idx = cam_idx[o].astype(np.int64)
    pt_idx = pt_idx[o].astype(np.int64)
    P = _camera_frame(cams_true, cam_idx, X_true[pt_idx])
    if not (P[:, 2] < -MIN_DEPTH * 0.5).all():
        raise AssertionError("generator emitted an observation behind its camera")
    px = _pixels(cams_true, cam_idx, None, P)
    del P
    px += rng.normal(0.0, pixel_sigma, px.shape)
    if outlier_frac > 0:
        out = rng.random(len(cam_idx)) < outlier_frac
        px[out] += rng.uniform(-outlier_px, outlier_px, (int(out.sum()), 2))
    # initial state: orientation perturbed by a right-multiplied rotation about the
    # camera's own centre and the centre moved by N(0, t_sigma) (with the BAL
    # parameterization P = R X + t, perturbing R at fixed t would swing the
    # centre about the world origin by |C| * angle)
    cams = cams_true.copy()
    delta = rng.normal(0.0, rot_sigma, (len(cams), 3))
    r0 = Rotation.from_rotvec(cams[:, 0:3])
    centre = -np.einsum("nji,nj->ni", r0.as_matrix(), cams[:, 3:6])
    r1 = r0 * Rotation.from_rotvec(delta)
    centre = centre + rng.normal(0.0, t_sigma, (len(cams), 3))
    cams[:, 0:3] = r1.as_rotvec()
    cams[:, 3:6] = -np.einsum("nij,nj->ni", r1.as_matrix(), centre)
    pts = X_true + rng.normal(0.0, pt_sigma, X_true.shape)
    return Problem(cams, pts, cam_idx, pt_idx, px, name=name)


def _cover_cameras(cams, X, cam_idx, pt_idx, n_cam, rng, tan_h=1.0, tan_v=1.0):
    """Give every camera at least one observation of a point it sees."""
    cnt = np.bincount(cam_idx, minlength=n_cam)
    extra_c, extra_p = [], []
    # an unobserved camera cannot duplicate a pair, so any visible point will do
    for c in np.flatnonzero(cnt == 0):
        Rc = Rotation.from_rotvec(cams[c, 0:3]).as_matrix()
        P = X @ Rc.T + cams[c, 3:6]
        vis = _visible(P, tan_h, tan_v)
        if vis.any():
            dist = np.where(vis, np.einsum("ni,ni->n", P, P), np.inf)
            extra_c.append(c)
            extra_p.append(int(np.argmin(dist)))
        else:
            # nothing in view (e.g. a camera on the city edge facing outwards):
            # turn it towards its nearest point and observe that one
            Rc = Rotation.from_rotvec(cams[c, 0:3]).as_matrix()
            C = -Rc.T @ cams[c, 3:6]
            j = int(np.argmin(np.einsum("ni,ni->n", X - C, X - C)))
            Rn = _frames(C[None], (X[j] - C)[None])
            cams[c, 0:3] = Rotation.from_matrix(Rn).as_rotvec()[0]
            cams[c, 3:6] = -Rotation.from_rotvec(cams[c, 0:3]).as_matrix() @ C
            extra_c.append(c)
            extra_p.append(j)
    if extra_c:
        cam_idx = np.concatenate([cam_idx, np.array(extra_c, dtype=np.int64)])
        pt_idx = np.concatenate([pt_idx, np.array(extra_p, dtype=np.int64)])
    return cam_idx, pt_idx


# ---------------------------------------------------------------------------
# C1 / C2: ring of cameras looking at the origin
# ---------------------------------------------------------------------------

def make_ring(n_cameras, n_points, extra_track_mean, seed=0, radius=10.0, name=None):
    """configs[0] (16 cams, 1000 pts, 2+Poisson(2)) and configs[1] (49 cams, 7776 pts, 2+Poisson(2.1))."""
    rng = np.random.default_rng(seed)
    ang = 2.0 * np.pi * np.arange(n_cameras) / n_cameras
    centers = np.stack([radius * np.cos(ang), radius * np.sin(ang), np.zeros(n_cameras)], axis=1)
    R = _frames(centers, -centers)
    cams = _cameras(centers, R, rng)
    X = rng.normal(0.0, 1.0, (n_points, 3))
    X = X[np.argsort(np.arctan2(X[:, 1], X[:, 0]), kind="stable")]
    P = np.einsum("cij,pj->pci", Rotation.from_rotvec(cams[:, 0:3]).as_matrix(), X) + cams[None, :, 3:6]
    vis = _visible(P)
    k = np.minimum(2 + rng.poisson(extra_track_mean, n_points), np.minimum(16, vis.sum(axis=1)))
    if (k < 2).any():
        raise RuntimeError("a point is visible from fewer than two cameras")
    keys = rng.random((n_points, n_cameras))
    keys[~vis] = np.inf
    cand = np.argsort(keys, axis=1)
    rows, cols, _ = _pick(cand, np.take_along_axis(vis, cand, axis=1), k)
    cam_idx, pt_idx = _cover_cameras(cams, X, cols, rows, n_cameras, rng)
    return _finish(name or f"ring{n_cameras}x{n_points}", cams, X, cam_idx, pt_idx, rng)


# ---------------------------------------------------------------------------
# C3: forward-moving trajectory through a corridor
# ---------------------------------------------------------------------------

def make_corridor(n_cameras=1200, n_points=160_000, seed=0, window=30, extra_track_mean=3.5,
                  half_width=5.0, half_height=5.0, name=None):
    """configs[2]: 1200 cams spaced 1 apart (yaw jitter 0.05), 160k corridor points.

    Points are uniform in a 10x10 cross-section (a 1-unit core around the
    trajectory kept clear) and observed by 2+Poisson(3.5) (mean 5.5) of the
    cameras up to ``window`` frames behind them that see them.
    """
    rng = np.random.default_rng(seed)
    yaw = rng.normal(0.0, 0.05, n_cameras)
    centers = np.stack([np.arange(n_cameras, dtype=np.float64), np.zeros(n_cameras),
                        np.zeros(n_cameras)], axis=1)
    fwd = np.stack([np.cos(yaw), np.sin(yaw), np.zeros(n_cameras)], axis=1)
    R = _frames(centers, fwd)
    cams = _cameras(centers, R, rng)
    X = np.empty((n_points, 3))
    X[:, 0] = rng.uniform(window * 0.5, n_cameras - 1 + window * 0.5, n_points)
    yz = rng.uniform(-1.0, 1.0, (n_points, 2)) * (half_width, half_height)
    core = (np.abs(yz[:, 0]) < 1.0) & (np.abs(yz[:, 1]) < 1.0)
    yz[core] *= 3.0
    X[:, 1:3] = yz
    X = X[np.argsort(X[:, 0], kind="stable")]
    base = np.floor(X[:, 0]).astype(np.int64)
    off = np.arange(1, window + 1)
    cand = base[:, None] - off[None, :] + 1
    inrange = (cand >= 0) & (cand < n_cameras)
    cand = np.clip(cand, 0, n_cameras - 1)
    Rm = Rotation.from_rotvec(cams[:, 0:3]).as_matrix()
    P = np.einsum("pcij,pj->pci", Rm[cand], X) + cams[cand, 3:6]
    vis = inrange & _visible(P)
    perm = np.argsort(rng.random(cand.shape), axis=1)
    cand = np.take_along_axis(cand, perm, axis=1)
    vis = np.take_along_axis(vis, perm, axis=1)
    k = np.minimum(2 + rng.poisson(extra_track_mean, n_points), vis.sum(axis=1))
    keep = k >= 2
    if not keep.all():  # drop the rare point no two cameras see
        X, cand, vis, k = X[keep], cand[keep], vis[keep], k[keep]
    rows, cols, _ = _pick(cand, vis, k)
    cam_idx, pt_idx = _cover_cameras(cams, X, cols, rows, n_cameras, rng)
    return _finish(name or f"corridor{n_cameras}x{len(X)}", cams, X, cam_idx, pt_idx, rng)


# ---------------------------------------------------------------------------
# C4: camera clusters on a sphere, heavy-tailed tracks, outliers
# ---------------------------------------------------------------------------

def make_mixed_tracks(n_cameras=72, n_points=400, seed=0, radius=10.0, name="mixed"):
    """Test problem with every track-length regime of the store: k = 1 (single
    observation), short tracks packed many to a warp-tile, and long tracks
    (k > 32) that span several sub-tiles.  Ring of cameras looking at the
    origin, points ~ N(0, 0.5^2 I), 1 px noise, the usual perturbation."""
    rng = np.random.default_rng(seed)
    ang = 2.0 * np.pi * np.arange(n_cameras) / n_cameras
    centers = np.stack([radius * np.cos(ang), radius * np.sin(ang), rng.uniform(-1, 1, n_cameras)], axis=1)
    R = _frames(centers, -centers)
    cams = _cameras(centers, R, rng)
    X = rng.normal(0.0, 0.5, (n_points, 3))
    P = np.einsum("cij,pj->pci", Rotation.from_rotvec(cams[:, 0:3]).as_matrix(), X) + cams[None, :, 3:6]
    vis = _visible(P)
    nvis = vis.sum(axis=1)
    kind = rng.random(n_points)
    k = np.where(kind < 0.2, 1, np.where(kind < 0.7, rng.integers(2, 13, n_points),
                                         rng.integers(33, n_cameras + 1, n_points)))
    k = np.minimum(k, nvis)
    if (k < 1).any():
        raise RuntimeError("a point is visible from no camera")
    keys = np.where(vis, rng.random((n_points, n_cameras)), 2.0)
    order = np.argsort(keys, axis=1)
    rows = np.repeat(np.arange(n_points), k)
    cols = order[rows, np.concatenate([np.arange(m) for m in k])]
    cam_idx, pt_idx = _cover_cameras(cams, X, cols.astype(np.int64), rows.astype(np.int64), n_cameras, rng)
    return _finish(name, cams, X, cam_idx, pt_idx, rng)


def make_clusters(n_cameras=1100, n_points=1_000_000, seed=0, n_clusters=8, radius=20.0,
                  p_geom=0.12, k_cap=200, outlier_frac=0.05, batch=25_000, name=None):
    """configs[3]: 1100 cams in 8 clusters on a radius-20 sphere, 1M points ~ N(0, 4 I).

    Track length 2+Geometric(0.12) capped at 200; each point belongs to one
    camera community (probability proportional to cluster size) and draws its
    cameras mostly from it, with Zipf-skewed camera popularity, which makes the
    per-camera observation counts very uneven.  5% of observations are
    outliers, uniform in +-50 px.
    """
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, n_clusters + 1)
    sizes = np.floor(n_cameras * w / w.sum()).astype(np.int64)
    sizes[0] += n_cameras - sizes.sum()
    dirs = rng.normal(size=(n_clusters, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    cl = np.repeat(np.arange(n_clusters), sizes)
    cdir = dirs[cl] + rng.normal(0.0, 0.15, (n_cameras, 3))
    cdir /= np.linalg.norm(cdir, axis=1, keepdims=True)
    centers = radius * cdir
    fwd = -cdir + rng.normal(0.0, 0.02, (n_cameras, 3))
    R = _frames(centers, fwd)
    cams = _cameras(centers, R, rng)
    within = np.concatenate([np.arange(s) for s in sizes])
    pop = 1.0 / (within + 1.0) ** 0.7
    X = rng.normal(0.0, 2.0, (n_points, 3))
    comm = rng.choice(n_clusters, size=n_points, p=sizes / sizes.sum())
    # spatial order inside a community: coarse morton code
    q = np.clip(((X[:, 0:2] + 8.0) * 4.0).astype(np.int64), 0, 63)
    X_order = np.lexsort((_morton2(q[:, 0], q[:, 1]), comm))
    X, comm = X[X_order], comm[X_order]
    k = np.minimum(2 + rng.geometric(p_geom, n_points), k_cap)
    Rm = Rotation.from_rotvec(cams[:, 0:3]).as_matrix()
    logw_in = np.log(pop).astype(np.float32)
    logw_out = (np.log(pop) + np.log(0.01)).astype(np.float32)
    rows_all, cams_all = [], []
    for a in range(0, n_points, batch):
        b = min(n_points, a + batch)
        Xb = X[a:b]
        P = np.einsum("cij,pj->pci", Rm, Xb) + cams[None, :, 3:6]
        vis = _visible(P)
        score = np.where(comm[a:b, None] == cl[None, :], logw_in[None, :], logw_out[None, :])
        score = score - np.log(-np.log(rng.random(score.shape, dtype=np.float32) + 1e-30)).astype(np.float32)
        score[~vis] = -np.inf
        kb = np.minimum(k[a:b], vis.sum(axis=1))
        if (kb < 2).any():
            raise RuntimeError("cluster point visible from fewer than two cameras")
        kmax = int(kb.max())
        top = np.argpartition(-score, kmax - 1, axis=1)[:, :kmax]
        order = np.argsort(-np.take_along_axis(score, top, axis=1), axis=1)
        top = np.take_along_axis(top, order, axis=1)
        take = np.arange(kmax)[None, :] < kb[:, None]
        r, c = np.nonzero(take)
        rows_all.append(r + a)
        cams_all.append(top[r, c])
    pt_idx = np.concatenate(rows_all)
    cam_idx = np.concatenate(cams_all)
    cam_idx, pt_idx = _cover_cameras(cams, X, cam_idx, pt_idx, n_cameras, rng)
    return _finish(name or f"clusters{n_cameras}x{n_points}", cams, X, cam_idx, pt_idx, rng,
                   outlier_frac=outlier_frac)


# ---------------------------------------------------------------------------
# C5: city grid, cameras on streets with random headings, facade points
# ---------------------------------------------------------------------------

def make_city(n_cameras=13_700, n_points=4_500_000, seed=0, extent=200.0, street=20.0,
              setback=3.0, max_range=60.0, extra_track_mean=4.5, n_cand=128, batch=100_000,
              name=None):
    """configs[4]: 13,700 cameras on the streets of a 200x200 city grid, 4.5M facade points.

    Cameras stand on street lines every 20 units with uniformly random heading
    (120 deg horizontal, 90 deg vertical field of view); points lie on the
    facades of the 10x10 building blocks.  Each point is observed by
    2+Poisson(4.5) distinct cameras within 60 units that see it, drawn from a
    random candidate sample of the surrounding cells (no occlusion model).
    """
    rng = np.random.default_rng(seed)
    n_lines = int(round(extent / street)) + 1
    horiz = rng.random(n_cameras) < 0.5
    line = rng.integers(0, n_lines, n_cameras) * street
    along = rng.uniform(0.0, extent, n_cameras)
    cx = np.where(horiz, along, line)
    cy = np.where(horiz, line, along)
    centers = np.stack([cx, cy, np.full(n_cameras, 1.5)], axis=1)
    cell = street
    ncell = int(np.ceil(extent / cell)) + 1
    ci = np.clip((cx / cell).astype(np.int64), 0, ncell - 1)
    cj = np.clip((cy / cell).astype(np.int64), 0, ncell - 1)
    corder = np.lexsort((_morton2(ci * 4 + (cx % cell / 5).astype(np.int64),
                                  cj * 4 + (cy % cell / 5).astype(np.int64)),))
    centers = centers[corder]
    ci, cj = ci[corder], cj[corder]
    yaw = rng.uniform(0.0, 2.0 * np.pi, n_cameras)
    # cameras on the outer streets look into the city, not out of it
    cxr, cyr = centers[:, 0], centers[:, 1]
    hx, hy = np.cos(yaw), np.sin(yaw)
    flip_x = ((cxr <= 0.0) & (hx < 0)) | ((cxr >= extent) & (hx > 0))
    flip_y = ((cyr <= 0.0) & (hy < 0)) | ((cyr >= extent) & (hy > 0))
    yaw = np.where(flip_x, np.pi - yaw, yaw)
    yaw = np.where(flip_y, -yaw, yaw)
    pitch = rng.normal(0.0, 0.05, n_cameras)
    fwd = np.stack([np.cos(yaw) * np.cos(pitch), np.sin(yaw) * np.cos(pitch), np.sin(pitch)], axis=1)
    R = _frames(centers, fwd)
    cams = _cameras(centers, R, rng)
    Rm = Rotation.from_rotvec(cams[:, 0:3]).as_matrix()
    # cameras bucketed by cell
    cell_id = ci * ncell + cj
    cam_by_cell = np.argsort(cell_id, kind="stable")
    cell_start = np.searchsorted(cell_id[cam_by_cell], np.arange(ncell * ncell + 1))
    cell_cnt = np.diff(cell_start)

    # facade points
    nb = int(round(extent / street))
    lo = setback
    hi = street - setback

    def facade(r, n):
        bi = r.integers(0, nb, n)
        bj = r.integers(0, nb, n)
        face = r.integers(0, 4, n)
        u = r.uniform(lo, hi, n)
        x0, y0 = bi * street, bj * street
        x = np.where(face == 0, x0 + lo, np.where(face == 1, x0 + hi, x0 + u))
        y = np.where(face == 2, y0 + lo, np.where(face == 3, y0 + hi, y0 + u))
        return np.stack([x, y, r.uniform(0.5, 15.0, n)], axis=1)

    reach = int(np.ceil(max_range / cell))
    tan_h, tan_v = np.tan(np.radians(60.0)), 1.0
    cos_h = np.cos(np.radians(52.0))      # 8 deg margin inside the 60 deg half-FOV
    tan_vm = np.tan(np.radians(30.0))     # 15 deg margin inside the 45 deg half-FOV
    cxy32 = centers[:, 0:2].astype(np.float32)
    hxy32 = np.stack([np.cos(yaw), np.sin(yaw)], axis=1).astype(np.float32)
    def one_batch(bi):
        # independent stream per batch: deterministic under any thread schedule
        brng = np.random.default_rng([seed, 7, bi])
        n = batch
        Xb = facade(brng, n)
        pi = np.clip((Xb[:, 0] / cell).astype(np.int64), 0, ncell - 1)
        pj = np.clip((Xb[:, 1] / cell).astype(np.int64), 0, ncell - 1)
        qi = pi[:, None] + brng.integers(-reach, reach + 1, (n, n_cand))
        qj = pj[:, None] + brng.integers(-reach, reach + 1, (n, n_cand))
        inside = (qi >= 0) & (qi < ncell) & (qj >= 0) & (qj < ncell)
        cid = np.where(inside, qi * ncell + qj, 0)
        cnt = np.where(inside, cell_cnt[cid], 0)
        pick = (brng.random((n, n_cand), dtype=np.float32) * np.maximum(cnt, 1)).astype(np.int64)
        cand = cam_by_cell[np.minimum(cell_start[cid] + pick, n_cameras - 1)].astype(np.int32)
        # cheap planar visibility test (float32) with margins inside the true
        # field of view; _finish re-checks every kept observation exactly
        dx = Xb[:, None, 0].astype(np.float32) - cxy32[cand, 0]
        dy = Xb[:, None, 1].astype(np.float32) - cxy32[cand, 1]
        dz = Xb[:, None, 2].astype(np.float32) - np.float32(1.5)
        r2 = dx * dx + dy * dy
        along_fwd = dx * hxy32[cand, 0] + dy * hxy32[cand, 1]
        vis = (inside & (cnt > 0) & (r2 <= np.float32(max_range ** 2)) & (along_fwd >= np.float32(2.0))
               & (along_fwd > np.float32(cos_h) * np.sqrt(r2))
               & (np.abs(dz) < np.float32(tan_vm) * along_fwd))
        # compact the first 32 visible candidates per point before de-duplicating
        width = 32
        rank = np.cumsum(vis, axis=1) - 1
        r, c = np.nonzero(vis & (rank < width))
        comp = np.full((n, width), -1, dtype=np.int32)
        comp[r, rank[r, c]] = cand[r, c]
        kb = 2 + brng.poisson(extra_track_mean, n)
        rows, cols, nvis = _pick(comp, comp >= 0, kb)
        good = nvis >= 2          # points fewer than two cameras see are dropped
        remap = np.cumsum(good) - 1
        sel = good[rows]
        return Xb[good], remap[rows[sel]], cols[sel].astype(np.int64), float(nvis.mean())

    from concurrent.futures import ThreadPoolExecutor
    n_batches = -(-int(n_points * 1.03) // batch) + 1
    Xs, rows_all, cams_all = [], [], []
    have = 0
    bi = 0
    with ThreadPoolExecutor(max_workers=8) as pool:
        while have < n_points:
            res = list(pool.map(one_batch, range(bi, bi + n_batches)))
            bi += n_batches
            for Xg, rows, cols, _ in res:
                if have >= n_points:
                    break
                take = min(len(Xg), n_points - have)
                sel = rows < take
                Xs.append(Xg[:take])
                rows_all.append(rows[sel] + have)
                cams_all.append(cols[sel])
                have += take
            n_batches = 2
    X = np.concatenate(Xs)
    pt_idx = np.concatenate(rows_all)
    cam_idx = np.concatenate(cams_all)
    # spatially coherent landmark order
    qx = np.clip((X[:, 0] * 2).astype(np.int64), 0, 0xFFFF)
    qy = np.clip((X[:, 1] * 2).astype(np.int64), 0, 0xFFFF)
    lorder = np.argsort(_morton2(qx, qy), kind="stable")
    inv = np.empty_like(lorder)
    inv[lorder] = np.arange(len(lorder))
    X = X[lorder]
    pt_idx = inv[pt_idx]
    cam_idx, pt_idx = _cover_cameras(cams, X, cam_idx, pt_idx, n_cameras, rng, tan_h, tan_v)
    return _finish(name or f"city{n_cameras}x{n_points}", cams, X, cam_idx, pt_idx, rng)


def make_config(name: str, scale: float = 1.0, seed: int = 0) -> Problem:
    """Generate BASELINE config ``c1``..``c5``; ``scale`` < 1 shrinks points (tests)."""
    s = scale
    if name == "c1":
        return make_ring(16, max(8, int(1000 * s)), 2.0, seed=seed, name="c1")
    if name == "c2":
        return make_ring(49, max(8, int(7776 * s)), 2.1, seed=seed, name="c2")
    if name in ("c3", "c3m64"):
        nc = max(40, int(1200 * s))
        return make_corridor(nc, max(16, int(160_000 * s)), seed=seed, name="c3")
    if name == "c4":
        return make_clusters(max(16, int(1100 * s)), max(16, int(1_000_000 * s)), seed=seed, name="c4")
    if name == "c5":
        nc = max(64, int(13_700 * s))
        ext = 200.0 * max(s, 0.09) ** 0.5
        return make_city(nc, max(64, int(4_500_000 * s)), seed=seed,
                         extent=max(60.0, round(ext / 20.0) * 20.0), name="c5")
    raise ValueError(f"unknown config {name!r}")
