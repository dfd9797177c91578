"""ctypes binding of libpoba (include/poba.h) and a thin device-context wrapper.

The library is built in-tree (``make`` / ``__graft_entry__.build()``) at
``paper_2204_12834_b200/lib/libpoba.so``.  There is no CPU fallback: if the
library or a CUDA device is missing every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POBA_LIB") or os.path.join(_HERE, "lib", "libpoba.so")  # POBA_LIB: A/B builds

POBA_OK, POBA_EINVAL, POBA_ENOTSPD, POBA_ENONFINITE, POBA_ECUDA, POBA_ENCCL, POBA_EVANISH, POBA_EPARSE = range(8)
OP_W, OP_WT, OP_U_INV, OP_V_INV, OP_U, OP_SCHUR, OP_WVW = range(7)
(READ_U0, READ_V0, READ_B_P, READ_B_L, READ_D_P, READ_D_L, READ_U, READ_V, READ_U_INV, READ_V_INV,
 READ_B_TILDE, READ_STORAGE) = range(12)

_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)

_SIGS = {
    "poba_last_error": (ctypes.c_char_p, []),
    "poba_version": (ctypes.c_int, []),
    "poba_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)]),
    "poba_nccl_unique_id": (ctypes.c_int, [_P]),
    "poba_create_sharded": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "poba_destroy": (ctypes.c_int, [_P]),
    "poba_local_group_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)]),
    "poba_local_group_destroy": (ctypes.c_int, [_P]),
    "poba_create_local": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "poba_set_problem": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I64P, _I64P, _DP]),
    "poba_problem_info": (ctypes.c_int, [_P, _I64P]),
    "poba_term_layout": (ctypes.c_int, [_P, _IP]),
    "poba_get_ordering": (ctypes.c_int, [_P, _I64P, _I64P, _I64P]),
    "poba_get_groups": (ctypes.c_int, [_P, ctypes.c_int64, _I64P, _I64P, _I64P, _I64P]),
    "poba_linearize": (ctypes.c_int, [_P, _DP, _DP, _I64P]),
    "poba_linearize_explicit": (ctypes.c_int, [_P, _DP, _DP, _DP]),
    "poba_damp": (ctypes.c_int, [_P, ctypes.c_double, ctypes.c_int]),
    "poba_series_solve": (ctypes.c_int, [_P, ctypes.c_double, ctypes.c_int, _DP, _IP, _IP, _DP]),
    "poba_series_apply": (ctypes.c_int, [_P, _DP, ctypes.c_int, _DP]),
    "poba_back_substitute": (ctypes.c_int, [_P, _DP, _DP, _IP]),
    "poba_cost": (ctypes.c_int, [_P, _DP, _DP, ctypes.c_int, _DP, _I64P]),
    "poba_set_points": (ctypes.c_int, [_P, _DP]),
    "poba_accept_points": (ctypes.c_int, [_P]),
    "poba_get_points": (ctypes.c_int, [_P, _DP]),
    "poba_get_points_all": (ctypes.c_int, [_P, _DP]),
    "poba_apply": (ctypes.c_int, [_P, ctypes.c_int, _DP, _DP]),
    "poba_read": (ctypes.c_int, [_P, ctypes.c_int, _DP]),
    "poba_time_terms": (ctypes.c_int, [_P, ctypes.c_int, _DP, _DP, _IP]),
    "poba_spectral_radius": (ctypes.c_int, [_P, _DP, ctypes.c_double, ctypes.c_int, _DP, _IP, _IP]),
    "poba_materialize": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64, _DP]),
    "poba_launch_count": (ctypes.c_int64, [_P]),
    "poba_stream": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "poba_shard_bounds": (ctypes.c_int, [ctypes.c_int64, _I64P, ctypes.c_int, _I64P]),
    "poba_schur_diagonal": (ctypes.c_int, [_P, _DP]),
    "poba_set_precision": (ctypes.c_int, [_P, ctypes.c_int]),
    "poba_cluster_cameras": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I64P, _I64P,
                                            ctypes.c_int64, _I64P, _I64P, _I64P]),
    "poba_set_dl": (ctypes.c_int, [_P, _DP]),
    "poba_series_solve_clustered": (ctypes.c_int, [_P, _I64P, ctypes.c_int, ctypes.c_double, ctypes.c_int, _DP,
                                                   _IP, _IP]),
    "poba_bal_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(_P)]),
    "poba_bal_info": (ctypes.c_int, [_P, _I64P]),
    "poba_bal_copy": (ctypes.c_int, [_P, _DP, _DP, _I64P, _I64P, _DP]),
    "poba_bal_free": (ctypes.c_int, [_P]),
    "poba_pcg": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, _DP,
                                _IP, _DP, _IP, _DP]),
}
PRECOND_SCHUR_JACOBI, PRECOND_SERIES = 1, 2
_ASSERT_MESSAGES = ("preconditioner is not positive definite", "reduced system is not positive definite")

EXPORTED = tuple(_SIGS)


def load():
    """Load libpoba.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libpoba is not built ({LIB_PATH} missing); run `make` or "
                                   "__graft_entry__.build() -- there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class PobaError(RuntimeError):
    """CUDA / NCCL failure inside libpoba."""


def _check(status):
    if status == POBA_OK:
        return
    msg = load().poba_last_error().decode(errors="replace")
    if status == POBA_ENOTSPD and msg.startswith(_ASSERT_MESSAGES):
        raise AssertionError(msg)  # the reference asserts these (solvers.py:47, 53)
    if status in (POBA_EINVAL, POBA_ENOTSPD, POBA_ENONFINITE, POBA_EVANISH):
        raise ValueError(msg)
    raise PobaError(f"libpoba status {status}: {msg}")


def _d(a):
    return a.ctypes.data_as(_DP) if a is not None else None


def _i64(a):
    return a.ctypes.data_as(_I64P) if a is not None else None


def _f64(a, shape=None):
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        out = out.reshape(shape)
    return out


_PINNED_MIN_BYTES = 4 << 20


def host_empty(shape) -> np.ndarray:
    """Uninitialised float64 host array for a large device download.

    Large results (Delta x_l, landmark positions: 108 MB at C5) are allocated in
    page-locked memory from PyTorch's caching host allocator, so the library's
    device-to-host copy lands with one DMA instead of staging through its pinned
    buffer and a host copy into freshly faulted pages.  The array owns the
    block (its base is the pinned tensor); dropping it returns the block to the
    allocator's cache, so the next call of the same size reuses it.
    """
    n = int(np.prod(shape))
    if n * 8 >= _PINNED_MIN_BYTES:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy().reshape(shape)
        except Exception:  # no usable page-locked allocator: plain pages, staged copy
            pass
    return np.empty(shape)


def shard_bounds(k_per_point, nranks: int) -> np.ndarray:
    """Landmark bounds of each rank's shard (host-only; same plan as sharded contexts)."""
    k = np.ascontiguousarray(k_per_point, dtype=np.int64)
    out = np.zeros(nranks + 1, dtype=np.int64)
    _check(load().poba_shard_bounds(len(k), _i64(k), int(nranks), _i64(out)))
    return out


def cluster_cameras(n_cam, n_pt, cam_idx, pt_idx, max_cluster_size):
    """Host-only covisibility clustering (clustering.py:49-101): (assignment, n_clusters, cut)."""
    ci = np.ascontiguousarray(cam_idx, dtype=np.int64)
    pi = np.ascontiguousarray(pt_idx, dtype=np.int64)
    out = np.empty(int(n_cam), dtype=np.int64)
    nc, cut = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(load().poba_cluster_cameras(int(n_cam), int(n_pt), len(ci), _i64(ci), _i64(pi), int(max_cluster_size),
                                       _i64(out), ctypes.byref(nc), ctypes.byref(cut)))
    return out, int(nc.value), int(cut.value)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().poba_nccl_unique_id(ctypes.cast(buf, _P)))
    return buf.raw


class LocalGroup:
    """In-process virtual ranks on one device (poba_local_group_create).

    Each rank's ``Device(rank=r, nranks=n, group=g)`` must be driven by its own
    thread (collectives meet at a host barrier); the group outlives them."""

    def __init__(self, nranks: int):
        self._lib = load()
        h = _P()
        _check(self._lib.poba_local_group_create(int(nranks), ctypes.byref(h)))
        self._h, self.nranks = h, int(nranks)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.poba_local_group_destroy(self._h)
            self._h = None


class Device:
    """One libpoba context: a problem's device-resident store and system."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None,
                 group: LocalGroup | None = None):
        lib = load()
        h = _P()
        if group is not None:
            _check(lib.poba_create_local(device, rank, nranks, group._h, ctypes.byref(h)))
            self._group = group  # keep the group alive while this context exists
        elif nranks > 1:
            idbuf = ctypes.create_string_buffer(nccl_id, 128)
            _check(lib.poba_create_sharded(device, rank, nranks, ctypes.cast(idbuf, _P), ctypes.byref(h)))
        else:
            _check(lib.poba_create(device, ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.rank, self.nranks = rank, nranks
        self.device = device
        self.precision = 64
        self.n_cam = self.n_pt = self.n_obs = 0

    def close(self):
        if getattr(self, "_h", None):
            self._lib.poba_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- K0 -------------------------------------------------------------------
    def set_problem(self, n_cam, n_pt, cam_idx, pt_idx, pixels=None):
        cam_idx = np.ascontiguousarray(cam_idx, dtype=np.int64)
        pt_idx = np.ascontiguousarray(pt_idx, dtype=np.int64)
        pix = None if pixels is None else _f64(pixels)
        _check(self._lib.poba_set_problem(self._h, int(n_cam), int(n_pt), len(cam_idx), _i64(cam_idx),
                                          _i64(pt_idx), _d(pix)))
        self.n_cam, self.n_pt, self.n_obs = int(n_cam), int(n_pt), len(cam_idx)

    def info(self) -> dict:
        v = np.zeros(16, dtype=np.int64)
        _check(self._lib.poba_problem_info(self._h, _i64(v)))
        keys = ("n_groups", "n_tiles", "n_chunks", "n_partials", "n_obs_local", "n_slots", "lm_lo", "lm_hi",
                "max_slots", "n_long", "device_bytes", "k_max", "n_cam", "n_pt", "n_obs", "rank")
        d = dict(zip(keys, (int(x) for x in v)))
        t = ctypes.c_int(0)
        _check(self._lib.poba_term_layout(self._h, ctypes.byref(t)))
        d["term_layout"] = "table" if t.value else "gather"
        return d

    def ordering(self):
        o = np.empty(self.n_obs, dtype=np.int64)
        c = np.empty(self.n_obs, dtype=np.int64)
        p = np.empty(self.n_obs, dtype=np.int64)
        _check(self._lib.poba_get_ordering(self._h, _i64(o), _i64(c), _i64(p)))
        return o, c, p

    def groups(self):
        n = np.zeros(1, dtype=np.int64)
        _check(self._lib.poba_get_groups(self._h, 0, _i64(n), None, None, None))
        g = int(n[0])
        k = np.empty(g, dtype=np.int64)
        s = np.empty(g, dtype=np.int64)
        m = np.empty(g, dtype=np.int64)
        _check(self._lib.poba_get_groups(self._h, g, _i64(n), _i64(k), _i64(s), _i64(m)))
        return k, s, m

    # ---- state / linearization -------------------------------------------------
    def set_points(self, points):
        _check(self._lib.poba_set_points(self._h, _d(_f64(points, (self.n_pt, 3)))))

    def get_points(self, base=None):
        if base is not None:
            out = np.array(base, dtype=np.float64, copy=True)
        else:  # a shard fills only its own rows
            out = np.zeros((self.n_pt, 3)) if self.nranks > 1 else host_empty((self.n_pt, 3))
        _check(self._lib.poba_get_points(self._h, _d(out)))
        return out

    def get_points_all(self):
        """Every landmark's point: a sharded context gathers the other ranks' rows
        (collective -- every rank calls it)."""
        out = host_empty((self.n_pt, 3))
        _check(self._lib.poba_get_points_all(self._h, _d(out)))
        return out

    def accept_points(self):
        _check(self._lib.poba_accept_points(self._h))

    def linearize(self, cams, points=None) -> int:
        bad = np.zeros(1, dtype=np.int64)
        pts = None if points is None else _f64(points, (self.n_pt, 3))
        _check(self._lib.poba_linearize(self._h, _d(_f64(cams, (self.n_cam, 9))), _d(pts), _i64(bad)))
        return int(bad[0])

    def linearize_explicit(self, jp, jl, res):
        _check(self._lib.poba_linearize_explicit(self._h, _d(_f64(jp, (self.n_obs, 2, 9))),
                                                 _d(_f64(jl, (self.n_obs, 2, 3))), _d(_f64(res, (self.n_obs, 2)))))

    def damp(self, lam, identity=False):
        _check(self._lib.poba_damp(self._h, float(lam), 1 if identity else 0))

    # ---- series / back-substitution / cost ------------------------------------------
    def series_solve(self, epsilon, max_order, want_ratios=False):
        dp = np.empty(9 * self.n_cam)
        order = ctypes.c_int(0)
        conv = ctypes.c_int(0)
        ratios = np.empty(max_order + 1) if want_ratios else None
        _check(self._lib.poba_series_solve(self._h, float(epsilon), int(max_order), _d(dp), ctypes.byref(order),
                                           ctypes.byref(conv), _d(ratios)))
        return dp, int(order.value), bool(conv.value), ratios

    def series_apply(self, v, order):
        out = np.empty(9 * self.n_cam)
        _check(self._lib.poba_series_apply(self._h, _d(_f64(v)), int(order), _d(out)))
        return out

    def set_precision(self, bits):
        """Block storage precision 64 or 32 (PoBA-32); invalidates the linearization."""
        _check(self._lib.poba_set_precision(self._h, int(bits)))
        self.precision = int(bits)

    def set_dl(self, d_l):
        """Override the landmark damping diagonal D_l (n_pt, 3) of the current linearization."""
        _check(self._lib.poba_set_dl(self._h, _d(_f64(d_l, (self.n_pt, 3)))))

    def series_solve_clustered(self, cluster_of_cam, n_clusters, epsilon, max_order):
        dp = np.empty(9 * self.n_cam)
        order, conv = ctypes.c_int(0), ctypes.c_int(0)
        cl = np.ascontiguousarray(cluster_of_cam, dtype=np.int64)
        _check(self._lib.poba_series_solve_clustered(self._h, _i64(cl), int(n_clusters), float(epsilon),
                                                     int(max_order), _d(dp), ctypes.byref(order), ctypes.byref(conv)))
        return dp, int(order.value), bool(conv.value)

    def schur_diagonal(self):
        out = np.empty((self.n_cam, 9, 9))
        _check(self._lib.poba_schur_diagonal(self._h, _d(out)))
        return out

    def pcg(self, precond, order, tol, max_iter, resume=False, want_history=False):
        """Device PCG; returns (delta_p, iterations, final_rel, converged, rel_history)."""
        dp = np.empty(9 * self.n_cam)
        it, conv = ctypes.c_int(0), ctypes.c_int(0)
        rel = ctypes.c_double(0.0)
        hist = np.zeros(max(int(max_iter), 1)) if want_history else None
        _check(self._lib.poba_pcg(self._h, int(precond), int(order), float(tol), int(max_iter), int(bool(resume)),
                                  _d(dp), ctypes.byref(it), ctypes.byref(rel), ctypes.byref(conv), _d(hist)))
        return dp, it.value, rel.value, bool(conv.value), hist

    def back_substitute(self, delta_p=None, want_delta_l=True):
        nz = ctypes.c_int(0)
        dl = None
        if want_delta_l:  # a shard fills only its own rows
            dl = np.zeros(3 * self.n_pt) if self.nranks > 1 else host_empty(3 * self.n_pt)
        dp = None if delta_p is None else _f64(delta_p)
        _check(self._lib.poba_back_substitute(self._h, _d(dp), _d(dl), ctypes.byref(nz)))
        return dl, bool(nz.value)

    def cost(self, cams, points=None, trial=False):
        c = ctypes.c_double(0.0)
        bad = np.zeros(1, dtype=np.int64)
        pts = None if points is None else _f64(points, (self.n_pt, 3))
        _check(self._lib.poba_cost(self._h, _d(_f64(cams, (self.n_cam, 9))), _d(pts), 1 if trial else 0,
                                   ctypes.byref(c), _i64(bad)))
        return float(c.value), int(bad[0])

    # ---- operators / read-back -------------------------------------------------------
    def apply(self, op, v):
        n_out = 3 * self.n_pt if op in (OP_WT, OP_V_INV) else 9 * self.n_cam
        out = np.zeros(n_out)
        _check(self._lib.poba_apply(self._h, int(op), _d(_f64(v)), _d(out)))
        return out

    def read(self, what):
        shapes = {READ_U0: (self.n_cam, 9, 9), READ_U: (self.n_cam, 9, 9), READ_U_INV: (self.n_cam, 9, 9),
                  READ_V0: (self.n_pt, 3, 3), READ_V: (self.n_pt, 3, 3), READ_V_INV: (self.n_pt, 3, 3),
                  READ_B_P: (9 * self.n_cam,), READ_B_L: (3 * self.n_pt,), READ_D_P: (self.n_cam, 9),
                  READ_D_L: (self.n_pt, 3), READ_B_TILDE: (9 * self.n_cam,)}
        if what == READ_STORAGE:
            shape = (self.n_obs, 2, 13)
        else:
            shape = shapes[what]
        out = np.zeros(shape)
        _check(self._lib.poba_read(self._h, int(what), _d(out)))
        return out

    def time_terms(self, reps):
        a = ctypes.c_double(0)
        b = ctypes.c_double(0)
        n = ctypes.c_int(0)
        _check(self._lib.poba_time_terms(self._h, int(reps), ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return float(a.value), float(b.value), int(n.value)

    def spectral_radius(self, v0, tol, max_iter):
        rho = ctypes.c_double(0)
        it = ctypes.c_int(0)
        conv = ctypes.c_int(0)
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        _check(self._lib.poba_spectral_radius(self._h, _d(v0), float(tol), int(max_iter), ctypes.byref(rho),
                                              ctypes.byref(it), ctypes.byref(conv)))
        return float(rho.value), int(it.value), bool(conv.value)

    def materialize(self, op, limit):
        """Dense matrix of a camera-space operator, built on the device."""
        dim = 9 * self.n_cam
        out = np.empty((dim, dim))
        _check(self._lib.poba_materialize(self._h, int(op), int(limit), _d(out)))
        return out.T  # the library writes column-major

    def launch_count(self) -> int:
        return int(self._lib.poba_launch_count(self._h))

    def stream_ptr(self) -> int:
        s = _P()
        _check(self._lib.poba_stream(self._h, ctypes.byref(s)))
        return int(s.value or 0)
