"""GPU PCG baselines (libpoba poba_pcg / poba_schur_diagonal) against the reference.

Golden values: tests/golden/pcg.npz, produced by the reference's own
solvers.schur_diagonal_blocks / pcg_schur_jacobi / pcg_power_series_preconditioner
and lm.run(solver="pcg" | "pcg-power") (tests/golden/make_golden.py).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_problem, load_golden

pytestmark = pytest.mark.gpu

PROBLEMS = {"c1": "c1", "noisy": "noisy4x60"}
INC_TOL = 1e-9
COST_TOL = 1e-8
# CG amplifies summation-order differences by ~kappa(S) over tens of iterations;
# a converged PCG step is itself only accurate to its 1e-6 residual tolerance,
# so converged solutions are compared at that level (short runs at INC_TOL)
PCG_TOL = 1e-5


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d else 1.0)


@pytest.fixture(scope="module")
def P():
    import paper_2204_12834_b200 as pkg
    return pkg


def systems(P, tag):
    p, _ = golden_problem(PROBLEMS[tag])
    z = load_golden("pcg")
    assert p.fingerprint() == str(z[f"{tag}_fingerprint"])
    lin = P.linearize(p)
    return z, [(f"{tag}_l{j}_", lin.damp(float(z[f"{tag}_l{j}_lam"]))) for j in range(2)]


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
def test_schur_diagonal_blocks(P, tag):
    z, syss = systems(P, tag)
    for pre, s in syss:
        got = P.schur_diagonal_blocks(s)
        assert got.shape == z[pre + "schur_diag"].shape
        assert rel(got, z[pre + "schur_diag"]) < 1e-11


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
def test_pcg_schur_jacobi(P, tag):
    z, syss = systems(P, tag)
    for pre, s in syss:
        rels = []
        rep = P.pcg_schur_jacobi(s, 1e-6, 500, callback=lambda it, x, r: rels.append(r))
        assert abs(rep.iterations - int(z[pre + "jac_iters"])) <= 1 and rep.converged == bool(z[pre + "jac_conv"])
        assert rel(rep.delta_p, z[pre + "jac_delta_p"]) < PCG_TOL
        n = min(len(rels), len(z[pre + "jac_rels"]), 8)
        np.testing.assert_allclose(rels[:n], z[pre + "jac_rels"][:n], rtol=1e-6)
        again = P.pcg_schur_jacobi(s, 1e-6, 500)  # no callback: one device call
        assert again.iterations == rep.iterations
        assert rel(again.delta_p, rep.delta_p) < 1e-14
        short = P.pcg_schur_jacobi(s, 1e-3, 3)
        assert short.iterations == int(z[pre + "jac3_iters"]) and short.converged == bool(z[pre + "jac3_conv"])
        assert rel(short.delta_p, z[pre + "jac3_delta_p"]) < INC_TOL


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
@pytest.mark.parametrize("m", [0, 2])
def test_pcg_power_series_preconditioner(P, tag, m):
    z, syss = systems(P, tag)
    for pre, s in syss:
        rep = P.pcg_power_series_preconditioner(s, m, 1e-6, 500)
        assert abs(rep.iterations - int(z[pre + f"pow{m}_iters"])) <= 1
        assert rel(rep.delta_p, z[pre + f"pow{m}_delta_p"]) < PCG_TOL


def test_generic_preconditioner_callable(P):
    """A plain Python preconditioner runs the reference loop on device operator passes."""
    z, syss = systems(P, "noisy")
    pre, s = syss[0]
    rep = P.pcg(s, lambda v: P.apply_series_inverse(s, v, 2), 1e-6, 500)
    assert abs(rep.iterations - int(z[pre + "pow2_iters"])) <= 1
    assert rel(rep.delta_p, z[pre + "pow2_delta_p"]) < PCG_TOL
    dev_pre = P.make_schur_jacobi_preconditioner(s)
    rep2 = P.pcg(s, dev_pre, 1e-6, 500)
    assert abs(rep2.iterations - int(z[pre + "jac_iters"])) <= 1


@pytest.mark.parametrize("tag", sorted(PROBLEMS))
@pytest.mark.parametrize("solver", ["pcg", "pcg-power"])
def test_lm_trace_pcg(P, tag, solver):
    p, _ = golden_problem(PROBLEMS[tag])
    z = load_golden("pcg")
    t = f"{tag}_lm_{solver.replace('-', '_')}"
    tr = P.run(p, P.LmConfig(solver=solver, max_outer_iterations=10, max_order=2))
    costs = np.array([i.cost for i in tr.iterations])
    want = z[t + "_cost"]
    assert len(costs) == len(want)
    assert np.all(np.abs(costs - want) <= COST_TOL * want)
    assert [i.accepted for i in tr.iterations] == z[t + "_accepted"].tolist()
    got_inner = [i.inner_iterations for i in tr.iterations][1:]
    assert all(abs(a - b) <= 1 for a, b in zip(got_inner, z[t + "_inner"].tolist()[1:]))
    assert [i.order_m for i in tr.iterations][1:] == z[t + "_order"].tolist()[1:]


def test_pcg_zero_rhs_and_delta_l(P):
    """Zero b_tilde returns (0, 0 iterations, converged); the PCG step feeds back-substitution."""
    z = load_golden("explicit")
    lin = P.assemble_from_observations(z["dec_cam_idx"], z["dec_pt_idx"], z["dec_jp"], z["dec_jl"],
                                       np.zeros_like(z["dec_res"]), 2, 3)
    s = lin.damp(1e-2)
    rep = P.pcg_schur_jacobi(s)
    assert rep.iterations == 0 and rep.converged and rep.final_relative_residual == 0.0
    assert not rep.delta_p.any()
    _, syss = systems(P, "c1")
    pre, s = syss[0]
    rep = P.pcg_schur_jacobi(s)
    dl = P.back_substitute(s, rep.delta_p)
    # joint residual of the damped normal equations (reference tests/test_power_series.py:181-190 analogue)
    r_l = s.apply_wt(rep.delta_p) + s.V.reshape(-1, 3, 3).__matmul__(dl.reshape(-1, 3, 1)).ravel() + s.b_l
    assert np.linalg.norm(r_l) <= 1e-8 * np.linalg.norm(s.b_l)
