"""CPU oracle for the PoBA hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's algorithm for the
power-series Schur solve and everything that feeds it (reference:
``/root/reference/pkg/src/powerba``).  It exists so that

  * ``tests/`` can check the CUDA path against it (parity),
  * ``__graft_entry__.smoke()`` can check one tiny CUDA invocation, and
  * ``bench.py`` can time it as the CPU baseline / the ``--impl reference`` arm.

Nothing in the product package (``paper_2204_12834_b200``) may import it.  The
product path runs on the GPU only and fails loudly without its CUDA library.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
fixtures in ``tests/golden/`` that were produced by importing the *reference
itself* (script: ``tests/golden/make_golden.py``), and against the reference
test-suite's own known-answer values (scalar series 2 - 2^-m, stop-criterion
arithmetic, pass counts, cost 12.5, ...).

Every function cites the reference file:line it restates.  Arithmetic follows
the reference's operation order (per-k-group einsum contractions in float64,
``np.add.at`` scatters in storage order, Cholesky -> inv(L) -> L^-T L^-1), so on
the golden fixtures the oracle agrees with the reference to the last few ulps.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial.transform import Rotation

POSE = 9
POINT = 3
# blocks.py:36-37 -- sqrt(diag) of the Marquardt scaling is clamped to [1e-6, 1e6]
CLAMP_LO = 1e-6
CLAMP_HI = 1e6
# blocks.py:40 and lm.py:110 -- slab length used by the reference's streaming loops
SLAB = 512
# camera.py:22
MIN_DEPTH = 1e-12


def _f64sum(spec, *ops):
    # blocks.py:45-47: every contraction accumulates in float64
    return np.einsum(spec, *ops, dtype=np.float64)


# ---------------------------------------------------------------------------
# observation ordering (blocks.py:362-372, 405-417, 83-87)
# ---------------------------------------------------------------------------

def canonical_order(cam_idx, pt_idx, n_points):
    """(order, cam_sorted, pt_sorted): lexsort by (k of landmark, landmark, camera).

    Restates ``blocks._sorted_observation_order`` (blocks.py:362-372).
    """
    cam_idx = np.asarray(cam_idx, dtype=np.int64)
    pt_idx = np.asarray(pt_idx, dtype=np.int64)
    track_len = np.bincount(pt_idx, minlength=n_points)
    if track_len.min() == 0:
        raise ValueError("every point must be observed at least once")
    perm = np.lexsort((cam_idx, pt_idx, track_len[pt_idx]))
    return perm, cam_idx[perm], pt_idx[perm]


@dataclass(frozen=True)
class KGroup:
    """One run of landmarks with equal track length k (blocks.py:50-58)."""
    k: int
    start: int
    n: int
    lm_ids: np.ndarray
    cam_ids: np.ndarray


def k_groups(cam_sorted, pt_sorted, n_points):
    """Restates ``blocks._build_groups`` (blocks.py:405-417)."""
    track_len = np.bincount(pt_sorted, minlength=n_points)
    out = []
    cursor = 0
    for k in np.unique(track_len):
        k = int(k)
        n = int(np.count_nonzero(track_len == k))
        span = n * k
        out.append(KGroup(k, cursor, n, pt_sorted[cursor:cursor + span:k].copy(),
                          cam_sorted[cursor:cursor + span].reshape(n, k).copy()))
        cursor += span
    return out


# ---------------------------------------------------------------------------
# camera model (camera.py:49-135, 160-166)
# ---------------------------------------------------------------------------

def rotations(rotvecs):
    """camera.py:49-51 (scipy from_rotvec().as_matrix())."""
    return Rotation.from_rotvec(np.atleast_2d(rotvecs)).as_matrix()


def project(cams, pts, pixels, jacobians):
    """Residual (and analytic Jacobians) of the 9-parameter BAL camera.

    Restates ``camera.evaluate`` (camera.py:67-135).  Returns (res, valid) or
    (res, j_pose (n,2,9), j_point (n,2,3), valid).  Invalid rows (|P_z| < 1e-12)
    are zeroed.
    """
    cams = np.atleast_2d(np.asarray(cams, dtype=np.float64))
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    n = cams.shape[0]
    R = rotations(cams[:, 0:3])
    f, k1, k2 = cams[:, 6], cams[:, 7], cams[:, 8]
    Pc = np.einsum("nij,nj->ni", R, pts) + cams[:, 3:6]
    depth = Pc[:, 2]
    ok = np.abs(depth) >= MIN_DEPTH
    dz = np.where(ok, depth, 1.0)
    p = -Pc[:, 0:2] / dz[:, None]
    s = np.einsum("ni,ni->n", p, p)
    d = 1.0 + s * (k1 + k2 * s)
    res = (f * d)[:, None] * p
    if pixels is not None:
        res = res - pixels
    res = np.where(ok[:, None], res, 0.0)
    if not jacobians:
        return res, ok

    iz = 1.0 / dz
    dp = np.zeros((n, 2, 3))
    dp[:, 0, 0] = -iz
    dp[:, 1, 1] = -iz
    dp[:, 0, 2] = Pc[:, 0] * iz * iz
    dp[:, 1, 2] = Pc[:, 1] * iz * iz
    g = (2.0 * k1 + 4.0 * k2 * s)[:, None] * p
    dd = np.zeros((n, 2, 2))
    dd[:, 0, 0] = d
    dd[:, 1, 1] = d
    dd += p[:, :, None] * g[:, None, :]
    dd *= f[:, None, None]
    A = dd @ dp
    skew = np.zeros((n, 3, 3))
    skew[:, 0, 1] = -pts[:, 2]
    skew[:, 0, 2] = pts[:, 1]
    skew[:, 1, 0] = pts[:, 2]
    skew[:, 1, 2] = -pts[:, 0]
    skew[:, 2, 0] = -pts[:, 1]
    skew[:, 2, 1] = pts[:, 0]
    jp = np.empty((n, 2, POSE))
    jp[:, :, 0:3] = A @ (-(R @ skew))
    jp[:, :, 3:6] = A
    jp[:, :, 6] = d[:, None] * p
    jp[:, :, 7] = (f * s)[:, None] * p
    jp[:, :, 8] = (f * s * s)[:, None] * p
    jl = A @ R
    jp[~ok] = 0.0
    jl[~ok] = 0.0
    return res, jp, jl, ok


def compose(rotvecs, deltas):
    """camera.py:160-166: log(R(w) Exp(delta)), canonical axis-angle."""
    r = Rotation.from_rotvec(np.atleast_2d(rotvecs)) * Rotation.from_rotvec(np.atleast_2d(deltas))
    return r.as_rotvec()


# ---------------------------------------------------------------------------
# linearization + damping (blocks.py:293-324, 333-352, 375-402, 164-192, 277-285)
# ---------------------------------------------------------------------------

@dataclass
class OracleLin:
    store: np.ndarray          # (n_obs, 2, 13) rows in canonical order
    order: np.ndarray
    cam_sorted: np.ndarray
    pt_sorted: np.ndarray
    groups: list
    n_cameras: int
    n_points: int
    U0: np.ndarray
    V0: np.ndarray
    b_p: np.ndarray
    b_l: np.ndarray
    D_p: np.ndarray
    D_l: np.ndarray
    n_invalid: int


def _reduce(store, cam_sorted, pt_sorted, order, n_cam, n_pt, n_invalid):
    """blocks.py:375-402: U0/V0/b_p/b_l via slab-wise np.add.at in storage order."""
    if np.bincount(cam_sorted, minlength=n_cam).min() == 0:
        raise ValueError("every camera must have at least one observation")
    groups = k_groups(cam_sorted, pt_sorted, n_pt)
    U0 = np.zeros((n_cam, POSE, POSE))
    V0 = np.zeros((n_pt, POINT, POINT))
    bp = np.zeros((n_cam, POSE))
    bl = np.zeros((n_pt, POINT))
    for a in range(0, store.shape[0], SLAB):
        s = slice(a, a + SLAB)
        jp = store[s, :, 0:9]
        jl = store[s, :, 9:12]
        r = store[s, :, 12]
        np.add.at(U0, cam_sorted[s], _f64sum("oai,oaj->oij", jp, jp))
        np.add.at(V0, pt_sorted[s], _f64sum("oai,oaj->oij", jl, jl))
        np.add.at(bp, cam_sorted[s], _f64sum("oai,oa->oi", jp, r))
        np.add.at(bl, pt_sorted[s], _f64sum("oai,oa->oi", jl, r))
    ii = np.arange(POSE)
    D_p = np.sqrt(np.clip(U0[:, ii, ii], CLAMP_LO ** 2, CLAMP_HI ** 2))
    ii = np.arange(POINT)
    D_l = np.sqrt(np.clip(V0[:, ii, ii], CLAMP_LO ** 2, CLAMP_HI ** 2))
    return OracleLin(store, order, cam_sorted, pt_sorted, groups, n_cam, n_pt,
                     U0, V0, bp.ravel(), bl.ravel(), D_p, D_l, n_invalid)


def linearize(cam_idx, pt_idx, pixels, cams, pts, precision=64):
    """blocks.py:293-324; precision=32 stores the blocks as float32 (PoBA-32) and every
    later sum reads the rounded values in float64 (blocks.py:42-47)."""
    cams = np.asarray(cams, dtype=np.float64)
    pts = np.asarray(pts, dtype=np.float64)
    n_cam, n_pt = cams.shape[0], pts.shape[0]
    order, cs, ps = canonical_order(cam_idx, pt_idx, n_pt)
    n = len(order)
    store = np.empty((n, 2, 13))
    bad = 0
    for a in range(0, n, SLAB):
        s = slice(a, a + SLAB)
        res, jp, jl, ok = project(cams[cs[s]], pts[ps[s]], np.asarray(pixels)[order[s]], True)
        bad += int(np.count_nonzero(~ok))
        store[s, :, 0:9] = jp
        store[s, :, 9:12] = jl
        store[s, :, 12] = res
    if precision == 32:
        store = store.astype(np.float32).astype(np.float64)
    return _reduce(store, cs, ps, order, n_cam, n_pt, bad)


def linearize_explicit(cam_idx, pt_idx, jp, jl, res, n_cam, n_pt, precision=64):
    """blocks.py:333-352 (assemble_from_observations)."""
    cam_idx = np.asarray(cam_idx, dtype=np.int64)
    pt_idx = np.asarray(pt_idx, dtype=np.int64)
    order, cs, ps = canonical_order(cam_idx, pt_idx, n_pt)
    store = np.empty((len(cam_idx), 2, 13))
    store[:, :, 0:9] = np.asarray(jp)[order]
    store[:, :, 9:12] = np.asarray(jl)[order]
    store[:, :, 12] = np.asarray(res)[order]
    if precision == 32:
        store = store.astype(np.float32).astype(np.float64)
    return _reduce(store, cs, ps, order, n_cam, n_pt, 0)


def spd_inverse(blocks, what):
    """blocks.py:277-285: Cholesky, inv(L), L^-T L^-1."""
    try:
        L = np.linalg.cholesky(blocks)
    except np.linalg.LinAlgError:
        raise ValueError(f"{what} blocks are not positive definite, assembly bug "
                         "or lambda too small") from None
    Li = np.linalg.inv(L)
    return np.einsum("pki,pkj->pij", Li, Li)


class OracleSystem:
    """Damped system at one (linearization, lambda); restates blocks.py:156-260."""

    def __init__(self, lin: OracleLin, lam: float, damping: str = "marquardt"):
        if lam < 0:
            raise ValueError("lambda must be non-negative")
        if damping not in ("marquardt", "identity"):
            raise ValueError(f"unknown damping mode {damping!r}")
        self.lin = lin
        self.lam = float(lam)
        Dp = np.ones_like(lin.D_p) if damping == "identity" else lin.D_p
        Dl = np.ones_like(lin.D_l) if damping == "identity" else lin.D_l
        self.D_p, self.D_l = Dp, Dl
        self.b_p, self.b_l = lin.b_p, lin.b_l
        self.U = lin.U0.copy()
        ii = np.arange(POSE)
        self.U[:, ii, ii] += lam * Dp ** 2
        self.V = lin.V0.copy()
        ii = np.arange(POINT)
        self.V[:, ii, ii] += lam * Dl ** 2
        self.U_inv = spd_inverse(self.U, "damped pose")
        self.V_inv = spd_inverse(self.V, "damped point")
        self.passes = {"w": 0, "wt": 0, "u_inv": 0, "v_inv": 0}
        self._bt = None

    @property
    def n_cameras(self):
        return self.lin.n_cameras

    @property
    def n_points(self):
        return self.lin.n_points

    def _views(self):
        for g in self.lin.groups:
            yield g, self.lin.store[g.start:g.start + g.n * g.k].reshape(g.n, g.k, 2, 13)

    def apply_w(self, v_l):
        """blocks.py:214-224."""
        v = np.asarray(v_l, dtype=np.float64).reshape(self.n_points, POINT)
        out = np.zeros((self.n_cameras, POSE))
        for g, blk in self._views():
            u = _f64sum("gkab,gb->gka", blk[..., 9:12], v[g.lm_ids])
            np.add.at(out, g.cam_ids, _f64sum("gkab,gka->gkb", blk[..., 0:9], u))
        self.passes["w"] += 1
        return out.ravel()

    def apply_wt(self, v_p):
        """blocks.py:226-236."""
        v = np.asarray(v_p, dtype=np.float64).reshape(self.n_cameras, POSE)
        out = np.zeros((self.n_points, POINT))
        for g, blk in self._views():
            u = _f64sum("gkab,gkb->gka", blk[..., 0:9], v[g.cam_ids])
            out[g.lm_ids] = _f64sum("gkab,gka->gb", blk[..., 9:12], u)
        self.passes["wt"] += 1
        return out.ravel()

    def apply_u_inv(self, v_p):
        """blocks.py:238-241."""
        self.passes["u_inv"] += 1
        return _f64sum("pij,pj->pi", self.U_inv,
                       np.asarray(v_p, dtype=np.float64).reshape(self.n_cameras, POSE)).ravel()

    def apply_v_inv(self, v_l):
        """blocks.py:243-246."""
        self.passes["v_inv"] += 1
        return _f64sum("pij,pj->pi", self.V_inv,
                       np.asarray(v_l, dtype=np.float64).reshape(self.n_points, POINT)).ravel()

    def apply_u(self, v_p):
        """blocks.py:248-250."""
        return _f64sum("pij,pj->pi", self.U,
                       np.asarray(v_p, dtype=np.float64).reshape(self.n_cameras, POSE)).ravel()

    def apply_schur(self, v_p):
        """blocks.py:252-254."""
        return self.apply_u(v_p) - self.apply_w(self.apply_v_inv(self.apply_wt(v_p)))

    def b_tilde(self):
        """blocks.py:256-260 (cached)."""
        if self._bt is None:
            self._bt = self.b_p - self.apply_w(self.apply_v_inv(self.b_l))
        return self._bt


def memory_account(n_obs, n_cam, n_pt, itemsize=8):
    """blocks.py:263-274 as a closed formula (tests/test_blocks.py:336-345)."""
    return (n_obs * 2 * 13 * itemsize + 3 * n_cam * 81 * 8 + 3 * n_pt * 9 * 8
            + 2 * (9 * n_cam + 3 * n_pt) * 8)


# ---------------------------------------------------------------------------
# power series (power_series.py:29-100)
# ---------------------------------------------------------------------------

def stop_test(x_i, x_prev, i, eps):
    """power_series.py:29-42."""
    if eps <= 0:
        raise ValueError("epsilon must be positive")
    if i < 1:
        raise ValueError("the criterion compares consecutive iterates, needs i >= 1")
    nx = np.linalg.norm(x_i)
    if nx == 0.0:
        raise ValueError("vanishing iterate norm with a nonzero right-hand side")
    return bool((i + 1) * np.linalg.norm(x_i - x_prev) / nx < eps)


def series_solve(system, eps=0.01, max_order=20, ratios=None):
    """power_series.py:45-77.  Returns (delta_p, order_used, converged).

    ``ratios`` (optional list) receives (i+1)||x_i - x_{i-1}|| / ||x_i|| per order.
    """
    if max_order < 0:
        raise ValueError("max_order must be non-negative")
    bt = system.b_tilde()
    if not np.any(bt):
        return np.zeros_like(bt), 0, True
    t = system.apply_u_inv(-bt)
    x = t.copy()
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite series iterate at order 0, assembly is broken")
    for i in range(1, max_order + 1):
        t = system.apply_u_inv(system.apply_w(system.apply_v_inv(system.apply_wt(t))))
        prev = x
        x = x + t
        if not np.all(np.isfinite(x)):
            raise ValueError(f"non-finite series iterate at order {i}, assembly is broken")
        if ratios is not None:
            nx = np.linalg.norm(x)
            ratios.append((i + 1) * np.linalg.norm(x - prev) / nx if nx else math.inf)
        if stop_test(x, prev, i, eps):
            return x, i, True
    return x, max_order, False


def back_sub(system, delta_p):
    """power_series.py:94-100: dx_l = -V^-1 (b_l + W^T dx_p)."""
    return -system.apply_v_inv(system.b_l + system.apply_wt(delta_p))


def series_apply(system, v, order):
    """power_series.py:80-91 (apply_series_inverse): x = sum_{i<=order} (U^-1 W V^-1 W^T)^i U^-1 v."""
    if order < 0:
        raise ValueError("order must be non-negative")
    t = system.apply_u_inv(np.asarray(v, dtype=np.float64))
    x = t.copy()
    for _ in range(order):
        t = system.apply_u_inv(system.apply_w(system.apply_v_inv(system.apply_wt(t))))
        x += t
    return x


# ---------------------------------------------------------------------------
# preconditioned CG baselines (solvers.py:30-118)
# ---------------------------------------------------------------------------

def schur_diagonal_blocks(system):
    """solvers.py:71-85: U_c - sum_{o in c} W_o V_l^-1 W_o^T, W_o = J_p^T J_l (9x3)."""
    M = system.U.copy()
    for g, blk in system._views():
        jp, jl = blk[..., 0:POSE], blk[..., POSE:POSE + POINT]
        w_obs = _f64sum("gkai,gkaj->gkij", jp, jl)
        tmp = _f64sum("gkij,gjl->gkil", w_obs, system.V_inv[g.lm_ids])
        np.add.at(M, g.cam_ids, -_f64sum("gkil,gkjl->gkij", tmp, w_obs))
    return M


def schur_jacobi(system):
    """solvers.py:88-95: block-Jacobi preconditioner from the exact 9x9 diagonal of S."""
    m_inv = spd_inverse(schur_diagonal_blocks(system), "Schur diagonal")

    def apply(v):
        return _f64sum("pij,pj->pi", m_inv, np.asarray(v).reshape(system.n_cameras, POSE)).ravel()
    return apply


def pcg(system, apply_preconditioner, tol=1e-6, max_iter=500):
    """solvers.py:30-64: PCG on S dx_p = -b_tilde.  Returns (delta_p, iterations, rel, converged, rels)."""
    rhs = -system.b_tilde()
    x = np.zeros_like(rhs)
    if not np.any(rhs):
        return x, 0, 0.0, True, []
    r = rhs.copy()
    z = apply_preconditioner(r)
    rz = float(r @ z)
    assert rz > 0, "preconditioner is not positive definite"
    rz0 = rz
    p = z
    rel = 1.0
    rels = []
    for it in range(1, max_iter + 1):
        sp = system.apply_schur(p)
        psp = float(p @ sp)
        assert psp > 0, "reduced system is not positive definite"
        alpha = rz / psp
        x = x + alpha * p
        r = r - alpha * sp
        z = apply_preconditioner(r)
        rz_new = float(r @ z)
        rel = np.sqrt(max(rz_new, 0.0) / rz0)
        rels.append(rel)
        if rel < tol:
            return x, it, rel, True, rels
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, max_iter, rel, False, rels


# ---------------------------------------------------------------------------
# spectral diagnostics (spectral.py:54-143)
# ---------------------------------------------------------------------------

def u_inv_sqrt_blocks(system):
    """spectral.py:46-51: blockwise symmetric inverse square roots of the damped U."""
    w, Q = np.linalg.eigh(system.U)
    if w.min() <= 0:
        raise ValueError("damped pose blocks must be positive definite")
    return _f64sum("pik,pk,pjk->pij", Q, 1.0 / np.sqrt(w), Q)


def estimate_spectral_radius(system, tol=1e-9, max_iter=10000, seed=0):
    """spectral.py:54-86: power iteration on U^-1/2 W V^-1 W^T U^-1/2; (value, iterations, converged)."""
    uis = u_inv_sqrt_blocks(system)

    def apply_sym(v):
        y = _f64sum("pij,pj->pi", uis, v.reshape(system.n_cameras, POSE)).ravel()
        y = system.apply_w(system.apply_v_inv(system.apply_wt(y)))
        return _f64sum("pij,pj->pi", uis, y.reshape(system.n_cameras, POSE)).ravel()

    rng = np.random.default_rng(seed)
    v = rng.standard_normal(system.n_cameras * POSE)
    v /= np.linalg.norm(v)
    est = 0.0
    for it in range(1, max_iter + 1):
        w = apply_sym(v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0, it, True
        new = float(v @ w)
        v = w / nw
        if abs(new - est) <= tol * max(abs(new), 1e-300):
            return new, it, True
        est = new
    return est, max_iter, False


def _dense(apply, dim):
    out = np.empty((dim, dim))
    e = np.zeros(dim)
    for j in range(dim):
        e[j] = 1.0
        out[:, j] = apply(e)
        e[j] = 0.0
    return out


def verify_error_bound(system, orders):
    """spectral.py:98-143: (rho, orders, bound, measured, ||U^-1||, ||b_tilde||) from dense factorizations."""
    orders = np.asarray(sorted(int(m) for m in orders))
    dim = system.n_cameras * POSE
    S = _dense(system.apply_schur, dim)
    bt = system.b_tilde()
    exact = np.linalg.solve(S, -bt)
    P = _dense(lambda v: system.apply_u_inv(system.apply_w(system.apply_v_inv(system.apply_wt(v)))), dim)
    rho = float(np.max(np.abs(np.linalg.eigvals(P))))
    u_inv_norm = float(np.linalg.norm(_dense(system.apply_u_inv, dim), 2))
    b_norm = float(np.linalg.norm(bt))
    bound = rho ** (orders + 1.0) / (1.0 - rho) * u_inv_norm * b_norm
    measured = np.array([np.linalg.norm(series_apply(system, -bt, int(m)) - exact) for m in orders])
    return rho, orders, bound, measured, u_inv_norm, b_norm


# ---------------------------------------------------------------------------
# PoST clustering (clustering.py:49-148)
# ---------------------------------------------------------------------------

def cluster_cameras(cam_idx, pt_idx, n_cam, max_cluster_size):
    """clustering.py:49-101: (assignment, n_clusters, sizes, cut_observations)."""
    from collections import Counter
    order = np.lexsort((cam_idx, pt_idx))
    ps, cs = np.asarray(pt_idx)[order], np.asarray(cam_idx)[order]
    bnd = np.flatnonzero(np.diff(ps)) + 1
    weights = Counter()
    for cams in np.split(cs, bnd):
        for i in range(len(cams)):
            for j in range(i + 1, len(cams)):
                weights[(int(cams[i]), int(cams[j]))] += 1
    parent = np.arange(n_cam)
    size = np.ones(n_cam, dtype=np.int64)

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a
    for (ci, cj), _ in sorted(weights.items(), key=lambda kv: (-kv[1], kv[0])):
        ra, rb = find(ci), find(cj)
        if ra == rb or size[ra] + size[rb] > max_cluster_size:
            continue
        keep, drop = min(ra, rb), max(ra, rb)
        parent[drop] = keep
        size[keep] += size[drop]
    roots = np.array([find(c) for c in range(n_cam)])
    ur = np.unique(roots)
    assignment = np.searchsorted(ur, roots)
    cut = sum(len(c) for c in np.split(assignment[cs], bnd) if np.unique(c).size > 1)
    return assignment, len(ur), np.bincount(assignment), int(cut)


def solve_clustered(lin, lam, assignment, n_clusters, eps, max_order):
    """clustering.py:104-148: per-cluster restricted systems (global D kept), series solved per cluster."""
    delta = np.zeros((lin.n_cameras, POSE))
    order_used, converged = 0, True
    cs, ps = lin.cam_sorted, lin.pt_sorted
    for c in range(n_clusters):
        cams = np.flatnonzero(assignment == c)
        cam_map = np.full(lin.n_cameras, -1)
        cam_map[cams] = np.arange(len(cams))
        mask = np.isin(cs, cams)
        kept = np.unique(ps[mask])
        lm_map = np.full(lin.n_points, -1)
        lm_map[kept] = np.arange(len(kept))
        rows = lin.store[mask]
        sub = linearize_explicit(cam_map[cs[mask]], lm_map[ps[mask]], rows[:, :, 0:9], rows[:, :, 9:12],
                                 rows[:, :, 12], len(cams), len(kept))
        sub.D_p = lin.D_p[cams]
        sub.D_l = lin.D_l[kept]
        dp, order, conv = series_solve(OracleSystem(sub, lam), eps, max_order)
        delta[cams] = dp.reshape(len(cams), POSE)
        order_used = max(order_used, order)
        converged = converged and conv
    return delta.ravel(), order_used, converged


# ---------------------------------------------------------------------------
# cost, retraction, LM loop (lm.py:107-144, 167-232)
# ---------------------------------------------------------------------------

def cost(cam_idx, pt_idx, pixels, cams, pts):
    """lm.py:107-119: 0.5 sum ||r||^2 in file order, slab-wise; (cost, n_invalid)."""
    total = 0.0
    bad = 0
    n = len(cam_idx)
    for a in range(0, n, SLAB):
        s = slice(a, a + SLAB)
        res, ok = project(cams[cam_idx[s]], pts[pt_idx[s]], pixels[s], False)
        total += 0.5 * float(np.einsum("oi,oi->", res, res))
        bad += int(np.count_nonzero(~ok))
    return total, bad


def retract(cams, pts, delta_p, delta_l):
    """lm.py:132-144."""
    dp = np.asarray(delta_p, dtype=np.float64).reshape(cams.shape[0], POSE)
    out = cams.copy()
    out[:, 0:3] = compose(cams[:, 0:3], dp[:, 0:3])
    out[:, 3:] += dp[:, 3:]
    return out, pts + np.asarray(delta_l, dtype=np.float64).reshape(-1, 3)


@dataclass
class OracleIter:
    iteration: int
    cost: float
    lam: float
    order_m: int
    accepted: bool
    n_invalid: int
    inner: int = 0


@dataclass
class OracleTrace:
    iterations: list = field(default_factory=list)
    converged: bool = False
    times: list = field(default_factory=list)


def lm_run(cam_idx, pt_idx, pixels, cams, pts, *, initial_lambda=1e-4,
           max_outer_iterations=50, relative_function_tolerance=1e-6,
           epsilon=0.01, max_order=20, lambda_decrease=2.0, lambda_increase=4.0,
           damping="marquardt", clock=None, solver="poba", cg_tolerance=1e-6, cg_max_iterations=500,
           precision=64, system_cls=None, lin0=None):
    """lm.py:167-232 for solver in {'poba', 'pcg', 'pcg-power'} (dispatch lm.py:147-164), precision=64.
    ``system_cls`` (default OracleSystem) may be ScaleOracleSystem for configuration-size runs;
    ``lin0`` optionally supplies the linearization at the initial state (already computed)."""
    import time
    clock = clock or time.perf_counter
    t0 = clock()
    cams = np.asarray(cams, dtype=np.float64).copy()
    pts = np.asarray(pts, dtype=np.float64).copy()
    c, bad = cost(cam_idx, pt_idx, pixels, cams, pts)
    if not np.isfinite(c):
        raise ValueError("initial cost is not finite")
    tr = OracleTrace()
    lam = initial_lambda
    tr.iterations.append(OracleIter(0, c, lam, 0, True, bad))
    tr.times.append(clock() - t0)
    lin = lin0
    for it in range(1, max_outer_iterations + 1):
        if lin is None:
            lin = linearize(cam_idx, pt_idx, pixels, cams, pts, precision)
        sys_ = (system_cls or OracleSystem)(lin, lam, damping)
        if solver == "poba":
            dp, order, _ = series_solve(sys_, epsilon, max_order)
            inner = order
        elif solver == "pcg":
            dp, inner, _, _, _ = pcg(sys_, schur_jacobi(sys_), cg_tolerance, cg_max_iterations)
            order = 0
        elif solver == "pcg-power":
            dp, inner, _, _, _ = pcg(sys_, lambda v: series_apply(sys_, v, max_order), cg_tolerance,
                                     cg_max_iterations)
            order = max_order
        else:
            raise ValueError(f"unknown solver {solver!r}")
        dl = back_sub(sys_, dp)
        if not dp.any() and not dl.any():
            tr.iterations.append(OracleIter(it, c, lam, order, True, lin.n_invalid, inner))
            tr.times.append(clock() - t0)
            tr.converged = True
            break
        tc, tp = retract(cams, pts, dp, dl)
        nc, tbad = cost(cam_idx, pt_idx, pixels, tc, tp)
        if nc < c:
            rel = (c - nc) / c if c > 0 else 0.0
            cams, pts, c = tc, tp, nc
            lam /= lambda_decrease
            lin = None
            tr.iterations.append(OracleIter(it, c, lam, order, True, tbad, inner))
            tr.times.append(clock() - t0)
            if rel < relative_function_tolerance:
                tr.converged = True
                break
        else:
            lam *= lambda_increase
            tr.iterations.append(OracleIter(it, c, lam, order, False, tbad, inner))
            tr.times.append(clock() - t0)
    return tr, cams, pts


# ---------------------------------------------------------------------------
# configuration-scale operator passes (C restatement, oracle/poba_term.c)
# ---------------------------------------------------------------------------

_TERM_LIB = None


def term_library():
    """ctypes handle of oracle/lib/libpoba_oracle.so (built by ``make oracle``);
    None if it is not built.  Test infrastructure, like the rest of this file."""
    global _TERM_LIB
    if _TERM_LIB is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libpoba_oracle.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        for name in ("oracle_apply_wt", "oracle_apply_w"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int64, P, P, P, ctypes.c_int64, P, P, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _TERM_LIB = lib
    return _TERM_LIB


class ScaleOracleSystem(OracleSystem):
    """OracleSystem whose W and W^T passes (blocks.py:214-236) run in the C
    restatement (oracle/poba_term.c, OpenMP over landmark runs / observation
    ranges) -- for parity checks at C4/C5 size.  U^-1, V^-1, b_tilde, the
    damping and the inverses are the numpy restatement above."""

    def __init__(self, lin: OracleLin, lam: float, damping: str = "marquardt", threads: int | None = None):
        super().__init__(lin, lam, damping)
        self._lib = term_library()
        if self._lib is None:
            raise RuntimeError("oracle/lib/libpoba_oracle.so is not built (make oracle)")
        self.threads = int(threads or self._lib.oracle_max_threads())
        self._store = np.ascontiguousarray(lin.store, dtype=np.float64)
        self._cs = np.ascontiguousarray(lin.cam_sorted, dtype=np.int64)
        self._ps = np.ascontiguousarray(lin.pt_sorted, dtype=np.int64)

    def _call(self, fn, n_out_rows, width, v):
        v = np.ascontiguousarray(v, dtype=np.float64).ravel()
        out = np.empty(n_out_rows * width)
        rc = fn(len(self._cs), self._store.ctypes.data, self._cs.ctypes.data, self._ps.ctypes.data, n_out_rows,
                v.ctypes.data, out.ctypes.data, self.threads)
        if rc:
            raise MemoryError("oracle pass failed")
        return out

    def apply_w(self, v_l):
        self.passes["w"] += 1
        return self._call(self._lib.oracle_apply_w, self.n_cameras, POSE, v_l)

    def apply_wt(self, v_p):
        self.passes["wt"] += 1
        return self._call(self._lib.oracle_apply_wt, self.n_points, POINT, v_p)
