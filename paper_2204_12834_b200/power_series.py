"""Truncated power-series solve of the reduced camera system, on the GPU.

Drop-in for the reference module ``powerba.power_series`` (reference
``pkg/src/powerba/power_series.py``).  With P = U^-1 W V^-1 W^T the order-m
approximation of S^-1 (-b_tilde) is built from t_0 = U^-1(-b_tilde),
t_i = P t_{i-1}, x(i) = x(i-1) + t_i, stopping once
(i+1) ||x(i) - x(i-1)|| / ||x(i)|| < epsilon.  The whole recurrence -- b_tilde,
every term, the norms and the stop test -- runs inside libpoba without host
round trips; only delta_p (9 n_cameras doubles) comes back.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["PowerSeriesResult", "stop_criterion", "series_terms", "power_series_solve",
           "apply_series_inverse", "back_substitute"]


@dataclass(frozen=True)
class PowerSeriesResult:
    """Pose-space solution of one truncated-series solve (power_series.py:20-26)."""

    delta_p: np.ndarray
    order_used: int
    converged: bool  # False when max_order ran out before the stop criterion


def stop_criterion(x_i: np.ndarray, x_prev: np.ndarray, i: int, epsilon: float) -> bool:
    """Host form of the inexactness test (power_series.py:29-42); the solver
    evaluates the same inequality on the device."""
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    if i < 1:
        raise ValueError("the criterion compares consecutive iterates, needs i >= 1")
    norm_x = np.linalg.norm(x_i)
    if norm_x == 0.0:
        raise ValueError("vanishing iterate norm with a nonzero right-hand side")
    return bool((i + 1) * np.linalg.norm(x_i - x_prev) / norm_x < epsilon)


def _device_system(system):
    from .blocks import DampedSystem
    if not isinstance(system, DampedSystem):
        raise TypeError("power_series_solve runs on the GPU and needs a paper_2204_12834_b200 "
                        "DampedSystem (from assemble / Linearization.damp); there is no CPU path")
    if system._b_l_override is not None:
        raise NotImplementedError("series solve with an overridden b_l is not supported on the device")
    system._activate()
    return system


def series_terms(system, rhs: np.ndarray):
    """Yield t_0 = U^-1 rhs, then t_i = (U^-1 W V^-1 W^T) t_{i-1} forever (power_series.py:45-50);
    each term is one fused device pass."""
    sys_ = _device_system(system)
    t = sys_.apply_u_inv(np.asarray(rhs, dtype=np.float64))
    while True:
        yield t
        t = sys_.apply_u_inv(sys_.apply_w_vinv_wt(t))


def power_series_solve(system, epsilon: float = 0.01, max_order: int = 20,
                       return_ratios: bool = False) -> PowerSeriesResult:
    """Solve S dx_p = -b_tilde by the truncated series (power_series.py:53-77).

    Same contract as the reference: ``max_order < 0`` and non-positive epsilon
    raise ValueError, a zero right-hand side returns (0, 0, True), exhaustion
    returns (x_m, m, False), and a non-finite iterate raises ValueError naming
    the order.  ``return_ratios`` additionally returns the per-order stop ratios.
    """
    if max_order < 0:
        raise ValueError("max_order must be non-negative")
    sys_ = _device_system(system)
    eps = float(epsilon)
    if not eps > 0:
        # the reference raises only once the criterion is evaluated (order >= 1
        # with a nonzero right-hand side)
        if not np.any(sys_.b_tilde()):
            res = PowerSeriesResult(np.zeros(sys_.n_pose_params), 0, True)
            return (res, None) if return_ratios else res
        if max_order >= 1:
            raise ValueError("epsilon must be positive")
        eps = 1.0
    with sys_._dp.lock:
        sys_._activate()
        dp, order, conv, ratios = sys_._dp.dev.series_solve(eps, max_order, want_ratios=return_ratios)
    c = sys_.counters
    if sys_._b_tilde is None:
        c.w += 1
        c.v_inv += 1
    if order or not conv:
        c.u_inv += order + 1
        c.w += order
        c.wt += order
        c.v_inv += order
    res = PowerSeriesResult(dp, order, conv)
    return (res, ratios) if return_ratios else res


def apply_series_inverse(system, v: np.ndarray, order: int) -> np.ndarray:
    """Fixed order-m series approximation of S^-1 applied to v (power_series.py:80-91)."""
    if order < 0:
        raise ValueError("order must be non-negative")
    sys_ = _device_system(system)
    with sys_._dp.lock:
        sys_._activate()
        out = sys_._dp.dev.series_apply(np.asarray(v, dtype=np.float64), order)
    sys_.counters.u_inv += order + 1
    sys_.counters.w += order
    sys_.counters.wt += order
    sys_.counters.v_inv += order
    return out


def back_substitute(system, delta_p: np.ndarray) -> np.ndarray:
    """dx_l = -V^-1 (b_l + W^T dx_p) (power_series.py:94-100)."""
    sys_ = _device_system(system)
    with sys_._dp.lock:
        sys_._activate()
        dl, _ = sys_._dp.dev.back_substitute(np.asarray(delta_p, dtype=np.float64))
    sys_.counters.wt += 1
    sys_.counters.v_inv += 1
    return dl
