"""Landmark-block store and matrix-free operators, device-resident.

Drop-in for the reference module ``powerba.blocks`` (reference
``pkg/src/powerba/blocks.py``): same entry points (``linearize``, ``assemble``,
``assemble_from_observations``, ``Linearization.damp``, ``memory_account``),
same ``DampedSystem`` surface (``apply_w``, ``apply_wt``, ``apply_u_inv``,
``apply_v_inv``, ``apply_u``, ``apply_schur``, ``b_tilde``, ``counters``) and the
same error messages.  Everything is computed by libpoba on the GPU; the
attributes the reference exposes as arrays (``U0``, ``V``, ``U_inv``, ``b_p``,
``store.storage_obs``, ...) are read back lazily from the device.
"""
from __future__ import annotations

import logging
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib

log = logging.getLogger(__name__)

POSE_DIM = 9
POINT_DIM = 3
BLOCK_COLS = POSE_DIM + POINT_DIM + 1  # 13

# blocks.py:36-37 -- clamp range of the Marquardt scaling sqrt(diag(J^T J))
DIAG_CLAMP_MIN = 1e-6
DIAG_CLAMP_MAX = 1e6


_PRECISION_DTYPES = {32: np.float32, 64: np.float64}


def _parse_precision(precision: int):
    """Block storage dtype (blocks.py:355-359); 32 = PoBA-32: fp32 blocks, fp64 reductions."""
    try:
        return _PRECISION_DTYPES[precision]
    except (KeyError, TypeError):
        raise ValueError(f"precision must be 32 or 64, got {precision}") from None


# ---------------------------------------------------------------------------
# device contexts bound to problems
# ---------------------------------------------------------------------------

class DeviceProblem:
    """libpoba context holding one problem's observation structure (K0)."""

    def __init__(self, cam_indices, pt_indices, pixels, n_cameras, n_points, device=0, rank=0, nranks=1,
                 nccl_id=None, group=None):
        self.dev = _lib.Device(device, rank, nranks, nccl_id, group)
        self.n_cameras, self.n_points = int(n_cameras), int(n_points)
        self.n_observations = len(cam_indices)
        self.dev.set_problem(n_cameras, n_points, cam_indices, pt_indices, pixels)
        self.cam_indices, self.pt_indices, self.pixels = cam_indices, pt_indices, pixels  # by reference
        self.generation = 0          # bumped by every (re)linearization
        self.active_system = None    # DampedSystem whose damping is on the device
        self.source = None           # what produced the current linearization
        self._ordering = None
        self._groups = None
        # One context is shared by every system built on this problem.  Each
        # activate-then-call sequence, and a whole lm.run, holds this lock, so
        # concurrent runs on one problem (the reference's
        # evalkit.run_benchmark(parallel=True), evalkit.py:162-196) serialise
        # on the device instead of overwriting each other's state mid-solve.
        self.lock = threading.RLock()

    def ordering(self):
        if self._ordering is None:
            self._ordering = self.dev.ordering()
        return self._ordering

    def groups(self):
        if self._groups is None:
            self._groups = self.dev.groups()
        return self._groups


def _signature(problem):
    return (id(problem.cam_indices), id(problem.pt_indices), id(problem.pixels),
            problem.cam_indices.shape, problem.n_cameras, problem.n_points)


_FULL_COPY_OBS = 2_000_000


def _snapshot(problem):
    """What a cached device store is validated against on the next lookup.

    Up to 2M observations: full copies of the observation arrays, compared
    element-wise.  Larger problems (C4, C5) are not copied; instead the arrays
    are made read-only for as long as the cache holds them, so an in-place edit
    raises at the write instead of silently reusing a stale device store (the
    flags are restored by ``invalidate``).  Arrays that are views of memory we
    cannot lock are validated by a full-content digest on every lookup."""
    arrs = (problem.cam_indices, problem.pt_indices, problem.pixels)
    if problem.cam_indices.shape[0] <= _FULL_COPY_OBS:
        return ("copy", tuple(np.array(a, copy=True) for a in arrs))
    locked = []
    for a in arrs:
        if isinstance(a, np.ndarray) and a.base is None and a.flags.writeable:
            a.flags.writeable = False
            locked.append(a)
    if all(isinstance(a, np.ndarray) and (a.base is None) and not a.flags.writeable for a in arrs):
        return ("locked", locked)
    return ("digest", _digest(arrs), locked)


def _digest(arrs):
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    for a in arrs:
        h.update(np.ascontiguousarray(a).view(np.uint8).reshape(-1))
    return h.digest()


def _same_snapshot(problem, snap):
    arrs = (problem.cam_indices, problem.pt_indices, problem.pixels)
    if snap[0] == "copy":
        return all(a.shape == b.shape and np.array_equal(a, b) for a, b in zip(arrs, snap[1]))
    if snap[0] == "locked":
        return all(not a.flags.writeable for a in arrs)
    return _digest(arrs) == snap[1]


def invalidate(problem) -> None:
    """Drop ``problem``'s cached device store (call after editing its observation
    arrays in place) and restore the write flags the cache set."""
    cached = getattr(problem, "_poba_device", None)
    if cached is None:
        return
    snap = cached[1]
    if snap[0] in ("locked", "digest"):
        for a in snap[-1]:
            a.flags.writeable = True
    try:
        object.__delattr__(problem, "_poba_device")
    except AttributeError:
        pass


def device_problem(problem, device: int = 0) -> DeviceProblem:
    """The (cached) device context of ``problem`` -- any object with the BalProblem arrays."""
    cached = getattr(problem, "_poba_device", None)
    sig = _signature(problem)
    if cached is not None and cached[0] == sig and _same_snapshot(problem, cached[1]):
        return cached[2]
    if cached is not None:
        invalidate(problem)
    dp = DeviceProblem(problem.cam_indices, problem.pt_indices, problem.pixels, problem.n_cameras,
                       problem.n_points, device=device)
    try:
        object.__setattr__(problem, "_poba_device", (sig, _snapshot(problem), dp))
    except (AttributeError, TypeError):
        pass
    return dp


# ---------------------------------------------------------------------------
# store view (reference LandmarkBlockStore, blocks.py:70-112)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class _Group:
    k: int
    obs_start: int
    n: int
    lm_ids: np.ndarray
    cam_ids: np.ndarray


@dataclass(frozen=True)
class LandmarkBlock:
    landmark_index: int
    camera_indices: np.ndarray
    data: np.ndarray  # (2k, 13)


class LandmarkBlockStore:
    """Host view of the device store: canonical (k, landmark, camera) order."""

    def __init__(self, lin: "Linearization"):
        self._lin = lin
        self._dp = lin._dp
        self.n_cameras = self._dp.n_cameras
        self.n_points = self._dp.n_points
        self._storage = None

    @property
    def cam_sorted(self):
        return self._dp.ordering()[1]

    @property
    def pt_sorted(self):
        return self._dp.ordering()[2]

    @property
    def order(self):
        return self._dp.ordering()[0]

    @property
    def dtype(self):
        return np.dtype(_PRECISION_DTYPES[self._lin.precision])

    @property
    def n_observations(self):
        return self._dp.n_observations

    @property
    def block_bytes(self) -> int:
        """sum over landmarks of 2k * 13 * itemsize, as the reference accounts it (blocks.py:97-100)."""
        return self.n_observations * 2 * BLOCK_COLS * self.dtype.itemsize

    @property
    def storage_obs(self):
        if self._storage is None:
            with self._dp.lock:
                self._lin._activate()
                self._storage = self._dp.dev.read(_lib.READ_STORAGE).astype(self.dtype, copy=False)
        return self._storage

    @property
    def groups(self):
        k, start, n = self._dp.groups()
        ps, cs = self.pt_sorted, self.cam_sorted
        out = []
        for kk, s, nn in zip(k.tolist(), start.tolist(), n.tolist()):
            out.append(_Group(kk, s, nn, ps[s:s + nn * kk:kk].copy(), cs[s:s + nn * kk].reshape(nn, kk).copy()))
        return out

    def group_views(self):
        st = self.storage_obs
        for g in self.groups:
            yield g, st[g.obs_start:g.obs_start + g.n * g.k].reshape(g.n, g.k, 2, BLOCK_COLS)

    def block(self, landmark_index: int) -> LandmarkBlock:
        ps = self.pt_sorted
        sel = np.flatnonzero(ps == landmark_index)
        off, k = int(sel[0]), len(sel)
        data = self.storage_obs[off:off + k].reshape(2 * k, BLOCK_COLS)
        return LandmarkBlock(landmark_index, self.cam_sorted[off:off + k].copy(), data)


# ---------------------------------------------------------------------------
# Linearization / DampedSystem
# ---------------------------------------------------------------------------

_STATE_COPY_BYTES = 32 << 20


_SAMPLE_ROWS = 4096


def _sample_index(n):
    """Evenly spaced rows (a strided view, so sampling costs no gather)."""
    return slice(0, n, max(1, n // _SAMPLE_ROWS))


def _frozen_state(cams, pts):
    """The state a Linearization re-linearizes from if another linearization
    replaced it on the device.  Cameras are always copied; points are copied up
    to 32 MB (every config but C5), larger point arrays are kept by reference
    with a sampled fingerprint that is re-checked before they are used again,
    so an in-place edit fails loudly instead of silently changing the system."""
    cams = np.array(cams, dtype=np.float64, copy=True)
    if pts.nbytes <= _STATE_COPY_BYTES:
        return cams, np.array(pts, dtype=np.float64, copy=True), None
    idx = _sample_index(len(pts))
    return cams, pts, (idx, pts[idx].copy())

class Linearization:
    """Device linearization (reference blocks.py:115-137); arrays read back lazily."""

    def __init__(self, dp: DeviceProblem, source, n_invalid: int, precision: int = 64):
        self._dp = dp
        self._source = source
        self.precision = int(precision)
        self.n_invalid = int(n_invalid)
        dp.generation += 1
        self._gen = dp.generation
        dp.source = source
        dp.active_system = None
        self.store = LandmarkBlockStore(self)
        self._cache = {}

    # re-run this linearization if another one replaced it on the device
    def _activate(self):
        dp = self._dp
        if dp.generation == self._gen:
            return
        kind = self._source[0]
        if kind == "state" and self._source[3] is not None:
            idx, vals = self._source[3]
            if not np.array_equal(self._source[2][idx], vals):
                raise ValueError("the points array this linearization was built from was modified in "
                                 "place; linearize the new state instead")
        dp.dev.set_precision(self.precision)
        if kind == "state":
            dp.dev.linearize(self._source[1], self._source[2])
        else:
            dp.dev.linearize_explicit(*self._source[1:])
        dp.generation += 1
        self._gen = dp.generation
        dp.active_system = None

    def _read(self, key, what):
        if key not in self._cache:
            with self._dp.lock:
                self._activate()
                self._cache[key] = self._dp.dev.read(what)
        return self._cache[key]

    @property
    def U0(self):
        return self._read("U0", _lib.READ_U0)

    @property
    def V0(self):
        return self._read("V0", _lib.READ_V0)

    @property
    def b_p(self):
        return self._read("b_p", _lib.READ_B_P)

    @property
    def b_l(self):
        return self._read("b_l", _lib.READ_B_L)

    @property
    def D_p(self):
        return self._read("D_p", _lib.READ_D_P)

    @property
    def D_l(self):
        return self._read("D_l", _lib.READ_D_L)

    @property
    def n_cameras(self) -> int:
        return self._dp.n_cameras

    @property
    def n_points(self) -> int:
        return self._dp.n_points

    def damp(self, lam: float, damping: str = "marquardt") -> "DampedSystem":
        return DampedSystem(self, lam, damping)


@dataclass
class OperatorCounts:
    """Block-operator pass counters (reference blocks.py:140-153)."""

    w: int = 0
    wt: int = 0
    u_inv: int = 0
    v_inv: int = 0

    def total(self) -> int:
        return self.w + self.wt + self.u_inv + self.v_inv

    def reset(self) -> None:
        self.w = self.wt = self.u_inv = self.v_inv = 0


class DampedSystem:
    """Damped reduced system at one (linearization, lambda), on the device.

    Reference blocks.py:156-260.  U/V blocks are damped and inverted by batched
    Cholesky kernels; the operator passes stream the device store.
    """

    def __init__(self, lin: Linearization, lam: float, damping: str = "marquardt"):
        if lam < 0:
            raise ValueError("lambda must be non-negative")
        if damping not in ("marquardt", "identity"):
            raise ValueError(f"unknown damping mode {damping!r}")
        self.lin = lin
        self.store = lin.store
        self.lam = float(lam)
        self.damping = damping
        self._dp = lin._dp
        with self._dp.lock:
            lin._activate()
            self._dp.dev.damp(self.lam, damping == "identity")
            self._dp.active_system = self
            self._gen = self._dp.generation
        self.counters = OperatorCounts()
        self._b_tilde = None
        self._cache = {}
        self._b_l_override = None

    def _activate(self):
        self.lin._activate()
        if self._dp.active_system is not self or self._gen != self._dp.generation:
            self._dp.dev.damp(self.lam, self.damping == "identity")
            self._dp.active_system = self
            self._gen = self._dp.generation

    def _read(self, key, what):
        if key not in self._cache:
            with self._dp.lock:
                self._activate()
                self._cache[key] = self._dp.dev.read(what)
        return self._cache[key]

    # -- attributes ------------------------------------------------------------
    @property
    def D_p(self):
        return np.ones_like(self.lin.D_p) if self.damping == "identity" else self.lin.D_p

    @property
    def D_l(self):
        return np.ones_like(self.lin.D_l) if self.damping == "identity" else self.lin.D_l

    @property
    def b_p(self):
        return self.lin.b_p

    @property
    def b_l(self):
        return self.lin.b_l if self._b_l_override is None else self._b_l_override

    @b_l.setter
    def b_l(self, value):
        # the reference lets tests overwrite b_l (tests/test_blocks.py:322-325)
        self._b_l_override = np.asarray(value, dtype=np.float64)
        self._b_tilde = None

    @property
    def U(self):
        return self._read("U", _lib.READ_U)

    @property
    def V(self):
        return self._read("V", _lib.READ_V)

    @property
    def U_inv(self):
        return self._read("U_inv", _lib.READ_U_INV)

    @property
    def V_inv(self):
        return self._read("V_inv", _lib.READ_V_INV)

    @property
    def n_cameras(self) -> int:
        return self._dp.n_cameras

    @property
    def n_points(self) -> int:
        return self._dp.n_points

    @property
    def n_pose_params(self) -> int:
        return POSE_DIM * self.n_cameras

    @property
    def n_point_params(self) -> int:
        return POINT_DIM * self.n_points

    # -- operator passes ------------------------------------------------------------
    def _op(self, op, v):
        with self._dp.lock:
            self._activate()
            return self._dp.dev.apply(op, v)

    def apply_w(self, v_l):
        """W v_l, landmark space to pose space (blocks.py:214-224)."""
        self.counters.w += 1
        return self._op(_lib.OP_W, np.asarray(v_l, dtype=np.float64).ravel())

    def apply_wt(self, v_p):
        """W^T v_p, pose space to landmark space (blocks.py:226-236)."""
        self.counters.wt += 1
        return self._op(_lib.OP_WT, np.asarray(v_p, dtype=np.float64).ravel())

    def apply_u_inv(self, v_p):
        self.counters.u_inv += 1
        return self._op(_lib.OP_U_INV, np.asarray(v_p, dtype=np.float64).ravel())

    def apply_v_inv(self, v_l):
        self.counters.v_inv += 1
        return self._op(_lib.OP_V_INV, np.asarray(v_l, dtype=np.float64).ravel())

    def apply_u(self, v_p):
        return self._op(_lib.OP_U, np.asarray(v_p, dtype=np.float64).ravel())

    def apply_w_vinv_wt(self, v_p):
        """W V^-1 W^T v_p in one pass of the fused series-term kernel (pose space to pose space)."""
        self.counters.w += 1
        self.counters.wt += 1
        self.counters.v_inv += 1
        return self._op(_lib.OP_WVW, np.asarray(v_p, dtype=np.float64).ravel())

    def apply_schur(self, v_p):
        """S v = (U - W V^-1 W^T) v, never forming S (blocks.py:252-254)."""
        return self._op(_lib.OP_SCHUR, np.asarray(v_p, dtype=np.float64).ravel())

    def b_tilde(self):
        """Reduced right-hand side b_p - W V^-1 b_l (cached), blocks.py:256-260."""
        if self._b_tilde is None:
            if self._b_l_override is not None:
                self._b_tilde = self.b_p - self.apply_w(self.apply_v_inv(self._b_l_override))
            else:
                with self._dp.lock:
                    self._activate()
                    self._b_tilde = self._dp.dev.read(_lib.READ_B_TILDE)
                self.counters.w += 1
                self.counters.v_inv += 1
        return self._b_tilde


def memory_account(system: DampedSystem) -> int:
    """The reference's analytic byte count of one damped system (blocks.py:263-274)."""
    n_p, n_l = system.n_cameras, system.n_points
    return (system.store.block_bytes + 3 * n_p * 81 * 8 + 3 * n_l * 9 * 8
            + 2 * (9 * n_p + 3 * n_l) * 8)


# ---------------------------------------------------------------------------
# assembly entry points
# ---------------------------------------------------------------------------

def linearize(problem, state=None, precision: int = 64, device: int = 0) -> Linearization:
    """Residuals + Jacobians at ``state`` packed into the device store (blocks.py:293-324)."""
    _parse_precision(precision)
    if state is None:
        state = problem
    cams = np.ascontiguousarray(state.camera_params, dtype=np.float64)
    pts = np.ascontiguousarray(state.points, dtype=np.float64)
    dp = device_problem(problem, device)
    with dp.lock:
        dp.dev.set_precision(precision)
        n_invalid = dp.dev.linearize(cams, pts)
        if n_invalid:
            log.warning("%d observation(s) had zero projected depth and were zeroed", n_invalid)
        return Linearization(dp, ("state",) + _frozen_state(cams, pts), n_invalid, precision)


def assemble(problem, state=None, lam: float = 1e-4, precision: int = 64,
             damping: str = "marquardt") -> DampedSystem:
    """linearize + damp in one call (blocks.py:327-330)."""
    return linearize(problem, state, precision).damp(lam, damping)


def assemble_from_observations(cam_indices, pt_indices, j_pose, j_point, residuals,
                               n_cameras: int, n_points: int, precision: int = 64,
                               device: int = 0) -> Linearization:
    """Pack a linearization from explicit per-observation arrays (blocks.py:333-352)."""
    _parse_precision(precision)
    cam_indices = np.asarray(cam_indices, dtype=np.int64)
    pt_indices = np.asarray(pt_indices, dtype=np.int64)
    dp = DeviceProblem(cam_indices, pt_indices, None, n_cameras, n_points, device=device)
    jp = np.ascontiguousarray(j_pose, dtype=np.float64)
    jl = np.ascontiguousarray(j_point, dtype=np.float64)
    r = np.ascontiguousarray(residuals, dtype=np.float64)
    dp.dev.set_precision(precision)
    dp.dev.linearize_explicit(jp, jl, r)
    return Linearization(dp, ("explicit", jp, jl, r), 0, precision)
