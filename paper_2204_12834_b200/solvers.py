"""Preconditioned CG baselines on the GPU operators.

Drop-in for the reference module ``powerba.solvers`` (reference
``pkg/src/powerba/solvers.py:30-118``) on the path the paper compares PoBA
against: CG on the reduced camera system S dx_p = -b_tilde, preconditioned
with the exact 9x9 diagonal blocks of S (Schur-Jacobi) or with the order-m
power series.  Every Schur product is one pass of the fused series-term kernel
(libpoba ``poba_pcg``); the CG recurrences, dot products and the relative
residual test follow ``pcg`` line by line.

A Python-callable preconditioner that is not one of the two device kinds is
honoured too: the loop then runs here, on device operator passes
(``DampedSystem.apply_schur``), exactly as the reference's ``pcg``.
"""
from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .power_series import _device_system, apply_series_inverse

__all__ = ["CgReport", "pcg", "schur_diagonal_blocks", "make_schur_jacobi_preconditioner",
           "pcg_schur_jacobi", "pcg_power_series_preconditioner", "materialize_schur", "dense_direct",
           "DENSE_DIM_LIMIT"]

# dense_direct refuses anything larger than this many pose parameters (solvers.py:17)
DENSE_DIM_LIMIT = 2000

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class CgReport:
    """Outcome of one conjugate-gradient solve (solvers.py:20-27)."""

    delta_p: np.ndarray
    iterations: int
    final_relative_residual: float
    converged: bool


class _DevicePreconditioner:
    """A preconditioner libpoba applies on the device (kind, series order)."""

    def __init__(self, system, kind: int, order: int = 0):
        self.system, self.kind, self.order = system, kind, order

    def __call__(self, v: np.ndarray) -> np.ndarray:
        """Apply outside a device PCG (convenience; the solve itself never calls this)."""
        if self.kind == _lib.PRECOND_SERIES:
            return apply_series_inverse(self.system, v, self.order)
        L = np.linalg.cholesky(schur_diagonal_blocks(self.system))
        eye = np.broadcast_to(np.eye(9), L.shape)
        L_inv = np.linalg.solve(L, eye)
        m_inv = np.einsum("pki,pkj->pij", L_inv, L_inv)
        return np.einsum("pij,pj->pi", m_inv, np.asarray(v, dtype=np.float64).reshape(-1, 9)).ravel()


def schur_diagonal_blocks(system) -> np.ndarray:
    """The 9x9 diagonal blocks of S: U_c - sum_l W_cl V_l^-1 W_cl^T (solvers.py:71-85)."""
    sys_ = _device_system(system)
    with sys_._dp.lock:
        sys_._activate()
        return sys_._dp.dev.schur_diagonal()


def make_schur_jacobi_preconditioner(system):
    """Block-Jacobi preconditioner from the true diagonal of S (solvers.py:88-95)."""
    sys_ = _device_system(system)
    with sys_._dp.lock:
        sys_._activate()
        sys_._dp.dev.schur_diagonal()  # raises ValueError if a block is not SPD, as the reference
    return _DevicePreconditioner(sys_, _lib.PRECOND_SCHUR_JACOBI)


def _pcg_device(sys_, pre: _DevicePreconditioner, tol, max_iter, callback):
    with sys_._dp.lock:
        sys_._activate()
        return _pcg_device_locked(sys_, pre, tol, max_iter, callback)


def _pcg_device_locked(sys_, pre, tol, max_iter, callback):
    dev = sys_._dp.dev
    if callback is None:
        dp, it, rel, conv, _ = dev.pcg(pre.kind, pre.order, tol, max_iter)
    else:  # one iteration per call so the callback sees every iterate
        dp, it, rel, conv, _ = dev.pcg(pre.kind, pre.order, tol, 0)
        while not conv and it < max_iter:
            dp, it, rel, conv, _ = dev.pcg(pre.kind, pre.order, tol, 1, resume=True)
            callback(it, dp, rel)
    if not conv and it >= max_iter and max_iter > 0:
        log.warning("PCG hit max_iter=%d with relative residual %.3e", max_iter, rel)
    c = sys_.counters
    c.w += it
    c.wt += it
    c.v_inv += it
    return CgReport(dp, it, rel, conv)


class _HostCg:
    """Preconditioned CG recurrences for a host-callable preconditioner
    (reference solvers.py:30-64): the Schur products are device passes
    (DampedSystem.apply_schur), the recurrences run here.  One ``advance``
    is one CG iteration; it returns the relative preconditioned residual
    sqrt(r.z / r0.z0)."""

    def __init__(self, sys_, precondition, rhs):
        self.sys_, self.precondition = sys_, precondition
        self.x = np.zeros_like(rhs)
        self.r = rhs.copy()
        self.z = precondition(self.r)
        self.rz = float(self.r @ self.z)
        assert self.rz > 0, "preconditioner is not positive definite"
        self.rz0 = self.rz
        self.p = self.z

    def advance(self) -> float:
        sp = self.sys_.apply_schur(self.p)
        curvature = float(self.p @ sp)
        assert curvature > 0, "reduced system is not positive definite"
        step = self.rz / curvature
        self.x = self.x + step * self.p
        self.r = self.r - step * sp
        self.z = self.precondition(self.r)
        rz_next = float(self.r @ self.z)
        rel = float(np.sqrt(max(rz_next, 0.0) / self.rz0))
        self.p = self.z + (rz_next / self.rz) * self.p
        self.rz = rz_next
        return rel


def pcg(system, apply_preconditioner, tol: float = 1e-6, max_iter: int = 500, callback=None) -> CgReport:
    """Preconditioned conjugate gradients on S dx_p = -b_tilde (solvers.py:30-64).

    The two device preconditioners (Schur-Jacobi, power series) run the whole
    solve in libpoba (``poba_pcg``); any other callable drives ``_HostCg``."""
    sys_ = _device_system(system)
    if isinstance(apply_preconditioner, _DevicePreconditioner) and apply_preconditioner.system is sys_:
        return _pcg_device(sys_, apply_preconditioner, tol, max_iter, callback)
    rhs = -sys_.b_tilde()
    if not np.any(rhs):
        return CgReport(np.zeros_like(rhs), 0, 0.0, True)
    cg = _HostCg(sys_, apply_preconditioner, rhs)
    rel = 1.0
    for it in range(1, max_iter + 1):
        rel = cg.advance()
        if callback is not None:
            callback(it, cg.x, rel)
        if rel < tol:
            return CgReport(cg.x, it, rel, True)
    log.warning("PCG hit max_iter=%d with relative residual %.3e", max_iter, rel)
    return CgReport(cg.x, max_iter, rel, False)


def pcg_schur_jacobi(system, tol: float = 1e-6, max_iter: int = 500, callback=None) -> CgReport:
    """CG preconditioned with the exact 9x9 diagonal blocks of S (solvers.py:98-102)."""
    sys_ = _device_system(system)
    return _pcg_device(sys_, _DevicePreconditioner(sys_, _lib.PRECOND_SCHUR_JACOBI), tol, max_iter, callback)


def pcg_power_series_preconditioner(system, order: int, tol: float = 1e-6, max_iter: int = 500,
                                    callback=None) -> CgReport:
    """CG preconditioned with the order-m series approximation of S^-1 (solvers.py:105-118)."""
    if order < 0:
        raise ValueError("order must be non-negative")
    sys_ = _device_system(system)
    return _pcg_device(sys_, _DevicePreconditioner(sys_, _lib.PRECOND_SERIES, order), tol, max_iter, callback)


def materialize_schur(system) -> np.ndarray:
    """S as a dense matrix (solvers.py:124-133), built on the device: one fused
    term pass per basis vector, one copy to the host (``poba_materialize``)."""
    sys_ = _device_system(system)
    with sys_._dp.lock:
        sys_._activate()
        return sys_._dp.dev.materialize(_lib.OP_SCHUR, _MATERIALIZE_LIMIT)


# the reference's materialize_schur has no size limit; this guards the device matrix
_MATERIALIZE_LIMIT = 40_000


def dense_direct(system) -> np.ndarray:
    """Solve S dx_p = -b_tilde by dense Cholesky; oracle-scale only (solvers.py:136-151).

    S is materialized on the device; the <= 2000 x 2000 factorization is host
    LAPACK, as in the reference."""
    import scipy.linalg
    sys_ = _device_system(system)
    dim = sys_.n_pose_params
    if dim > DENSE_DIM_LIMIT:
        raise ValueError(f"dense solve refused: {dim} pose parameters exceeds limit {DENSE_DIM_LIMIT}")
    try:
        chol = scipy.linalg.cho_factor(materialize_schur(sys_))
    except np.linalg.LinAlgError as exc:
        raise ValueError(f"materialized reduced system is not SPD: {exc}") from None
    return scipy.linalg.cho_solve(chol, -sys_.b_tilde())
