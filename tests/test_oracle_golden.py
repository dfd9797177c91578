"""Pin the CPU oracle (oracle/poba_oracle.py) to the reference.

Two kinds of pins, both CPU-only:
  * golden fixtures produced by running the reference itself
    (tests/golden/make_golden.py), compared at the last-few-ulps level;
  * the reference test-suite's own known-answer values
    (reference pkg/tests/test_power_series.py, test_lm.py, test_blocks.py).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_problem, load_golden
from oracle import poba_oracle as O

FIXTURES = ["rand3x5", "noisy4x60", "rig49", "c1", "c2", "mixed"]


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d else 1.0)


@pytest.mark.parametrize("name", FIXTURES)
def test_ordering_bit_exact(name):
    p, z = golden_problem(name)
    order, cs, ps = O.canonical_order(p.cam_indices, p.pt_indices, p.n_points)
    assert np.array_equal(order, z["order"])
    assert np.array_equal(cs, z["cam_sorted"]) and np.array_equal(ps, z["pt_sorted"])
    g = O.k_groups(cs, ps, p.n_points)
    assert [x.k for x in g] == z["group_k"].tolist()
    assert [x.start for x in g] == z["group_start"].tolist()
    assert [x.n for x in g] == z["group_n"].tolist()


@pytest.mark.parametrize("name", FIXTURES)
def test_linearization_matches_reference(name):
    p, z = golden_problem(name)
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    if "storage" in z:
        assert np.abs(lin.store - z["storage"]).max() <= 1e-12 * np.abs(z["storage"]).max()
    for key in ("U0", "V0", "b_p", "b_l", "D_p", "D_l"):
        assert rel(getattr(lin, key), z[key]) < 1e-13, key
    assert lin.n_invalid == int(z["n_invalid"])


@pytest.mark.parametrize("name", FIXTURES)
def test_series_and_back_substitution_match_reference(name):
    p, z = golden_problem(name)
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    j = 0
    while f"lam{j}" in z:
        s = O.OracleSystem(lin, float(z[f"lam{j}"]))
        assert rel(s.b_tilde(), z[f"sys{j}_b_tilde"]) < 1e-12
        i = 0
        while f"sys{j}_solve{i}_eps" in z:
            pre = f"sys{j}_solve{i}_"
            dp, order, conv = O.series_solve(s, float(z[pre + "eps"]), int(z[pre + "m"]))
            assert order == int(z[pre + "order"]) and conv == bool(z[pre + "converged"])
            assert rel(dp, z[pre + "delta_p"]) < 1e-11
            assert rel(O.back_sub(s, dp), z[pre + "delta_l"]) < 1e-11
            i += 1
        j += 1


@pytest.mark.parametrize("name", FIXTURES)
def test_cost_matches_reference(name):
    p, z = golden_problem(name)
    c, bad = O.cost(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    want_c, want_bad = z["cost0"]
    assert abs(c - want_c) <= 1e-13 * want_c and bad == int(want_bad)


@pytest.mark.parametrize("name,tag,kw", [
    ("rand3x5", "lm_poba", {}),
    ("noisy4x60", "lm_poba", {}),
    ("c1", "lm_c1", dict(max_outer_iterations=10, max_order=32)),
    ("c2", "lm_c2", dict(max_outer_iterations=20, max_order=32, epsilon=1e-6)),
    ("mixed", "lm_mixed", dict(max_outer_iterations=15, max_order=20)),
])
def test_lm_trace_matches_reference(name, tag, kw):
    p, z = golden_problem(name)
    tr, _, _ = O.lm_run(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points, **kw)
    costs = np.array([i.cost for i in tr.iterations])
    assert len(costs) == len(z[tag + "_cost"])
    assert np.allclose(costs, z[tag + "_cost"], rtol=1e-10, atol=0)
    assert [i.accepted for i in tr.iterations] == z[tag + "_accepted"].tolist()
    assert [i.order_m for i in tr.iterations] == z[tag + "_order"].tolist()
    assert [i.lam for i in tr.iterations] == z[tag + "_lam"].tolist()


def test_rig49_end_to_end_golden():
    """Reference criterion 6 golden: poba final cost 7584.4992 (pkg/test_output.txt:19)."""
    p, z = golden_problem("rig49")
    tr, _, _ = O.lm_run(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    assert round(tr.iterations[-1].cost, 4) == 7584.4992
    assert abs(tr.iterations[-1].cost - z["lm_poba_cost"][-1]) <= 1e-10 * z["lm_poba_cost"][-1]


def test_explicit_systems_match_reference():
    z = load_golden("explicit")
    for j in range(4):
        pre = f"e{j}_"
        lin = O.linearize_explicit(z[pre + "cam_idx"], z[pre + "pt_idx"], z[pre + "jp"],
                                   z[pre + "jl"], z[pre + "res"], int(z[pre + "n_cam"]),
                                   int(z[pre + "n_pt"]))
        for key in ("U0", "V0", "b_p", "b_l", "D_p", "D_l"):
            assert rel(getattr(lin, key), z[pre + key]) < 1e-14, key
        s = O.OracleSystem(lin, float(z[pre + "lam"]))
        i = 0
        while f"{pre}sys_solve{i}_eps" in z:
            q = f"{pre}sys_solve{i}_"
            dp, order, conv = O.series_solve(s, float(z[q + "eps"]), int(z[q + "m"]))
            assert order == int(z[q + "order"]) and conv == bool(z[q + "converged"])
            assert rel(dp, z[q + "delta_p"]) < 1e-12
            i += 1
    lin = O.linearize_explicit(z["dec_cam_idx"], z["dec_pt_idx"], z["dec_jp"], z["dec_jl"],
                               z["dec_res"], 2, 3)
    s = O.OracleSystem(lin, 1e-2)
    dp, order, conv = O.series_solve(s, 1e-12)
    assert order == 1 and conv and np.array_equal(dp, z["dec_delta_p"])
    assert np.array_equal(dp, z["dec_u_inv_minus_bt"])


# --- known-answer values from the reference's own unit tests -----------------

class _Mini:
    """Dense duck-typed system (reference tests/helpers.py:255-293 restated)."""

    def __init__(self, U, W, V, b_p, b_l):
        self.U, self.W, self.V = (np.atleast_2d(np.asarray(a, float)) for a in (U, W, V))
        self.b_p, self.b_l = np.atleast_1d(np.asarray(b_p, float)), np.atleast_1d(np.asarray(b_l, float))
        self.Ui, self.Vi = np.linalg.inv(self.U), np.linalg.inv(self.V)

    def apply_u_inv(self, v): return self.Ui @ v
    def apply_v_inv(self, v): return self.Vi @ v
    def apply_w(self, v): return self.W @ v
    def apply_wt(self, v): return self.W.T @ v
    def b_tilde(self): return self.b_p - self.W @ (self.Vi @ self.b_l)


def test_scalar_series_is_exact():
    # reference tests/test_power_series.py:23-46: x(m) = 2 - 0.5^m exactly
    for m in (0, 1, 5, 20):
        dp, order, conv = O.series_solve(_Mini(1.0, 0.5, 0.5, -1.0, 0.0), 1e-300, m)
        assert float(dp[0]) == 2.0 - 0.5 ** m and order == m and not conv


def test_stop_criterion_arithmetic():
    # reference tests/test_power_series.py:50-55
    assert O.stop_test(np.array([1.0, 0.0]), np.array([1.0, 0.004]), 1, 0.01)
    assert not O.stop_test(np.array([1.0, 0.0]), np.array([1.0, 0.004]), 3, 0.01)
    with pytest.raises(ValueError, match="positive"):
        O.stop_test(np.ones(2), np.ones(2), 1, 0.0)
    with pytest.raises(ValueError, match="vanishing"):
        O.stop_test(np.zeros(2), np.ones(2), 1, 0.01)


def test_zero_rhs_and_errors():
    dp, order, conv = O.series_solve(_Mini(np.eye(2), np.zeros((2, 2)), np.eye(2), np.zeros(2), np.zeros(2)))
    assert order == 0 and conv and not dp.any()
    with pytest.raises(ValueError, match="max_order"):
        O.series_solve(_Mini(1.0, 0.5, 0.5, -1.0, 0.0), max_order=-1)
    with pytest.raises(ValueError, match="non-finite series iterate at order 0"):
        O.series_solve(_Mini(1.0, 0.5, 0.5, np.nan, 0.0))
    with np.errstate(over="ignore"), pytest.raises(ValueError, match="order 1"):
        O.series_solve(_Mini(1.0, 1e200, 1.0, -1.0, 0.0))


def test_single_residual_cost():
    # reference tests/test_lm.py:25-27: cost 12.5
    c, bad = O.cost(np.array([0]), np.array([0]), np.array([[-3.0, -4.0]]),
                    np.array([[0, 0, 0, 0, 0, 0, 1.0, 0, 0]]), np.array([[0.0, 0.0, -1.0]]))
    assert c == 12.5 and bad == 0


def test_pass_counts():
    # reference tests/test_power_series.py:153-162: (w, wt, v_inv, u_inv) = (m, m, m, m+1)
    z = load_golden("explicit")
    lin = O.linearize_explicit(z["e3_cam_idx"], z["e3_pt_idx"], z["e3_jp"], z["e3_jl"], z["e3_res"],
                               int(z["e3_n_cam"]), int(z["e3_n_pt"]))
    s = O.OracleSystem(lin, 1e-2)
    s.b_tilde()
    s.passes = dict.fromkeys(s.passes, 0)
    O.series_solve(s, 1e-300, 6)
    assert (s.passes["w"], s.passes["wt"], s.passes["v_inv"], s.passes["u_inv"]) == (6, 6, 6, 7)


# -- PCG baselines (reference solvers.py:30-118), pinned by tests/golden/pcg.npz ----------

PCG_PROBLEMS = {"c1": "c1", "noisy": "noisy4x60"}


@pytest.mark.parametrize("tag", sorted(PCG_PROBLEMS))
def test_pcg_baselines_match_reference(tag):
    p, _ = golden_problem(PCG_PROBLEMS[tag])
    z = load_golden("pcg")
    assert p.fingerprint() == str(z[f"{tag}_fingerprint"])
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    for j in range(2):
        pre = f"{tag}_l{j}_"
        s = O.OracleSystem(lin, float(z[pre + "lam"]))
        assert rel(O.schur_diagonal_blocks(s), z[pre + "schur_diag"]) < 1e-12
        x, it, r, conv, rels = O.pcg(s, O.schur_jacobi(s), 1e-6, 500)
        assert it == int(z[pre + "jac_iters"]) and conv == bool(z[pre + "jac_conv"])
        assert rel(x, z[pre + "jac_delta_p"]) < 1e-10
        np.testing.assert_allclose(rels, z[pre + "jac_rels"], rtol=1e-6)
        for m in (0, 2):
            x, it, r, conv, _ = O.pcg(s, lambda v: O.series_apply(s, v, m), 1e-6, 500)
            assert it == int(z[pre + f"pow{m}_iters"])
            assert rel(x, z[pre + f"pow{m}_delta_p"]) < 1e-10
        x, it, r, conv, _ = O.pcg(s, O.schur_jacobi(s), 1e-3, 3)
        assert it == int(z[pre + "jac3_iters"]) and conv == bool(z[pre + "jac3_conv"])
        assert rel(x, z[pre + "jac3_delta_p"]) < 1e-10


@pytest.mark.parametrize("tag", sorted(PCG_PROBLEMS))
@pytest.mark.parametrize("solver", ["pcg", "pcg-power"])
def test_pcg_lm_trace_matches_reference(tag, solver):
    p, _ = golden_problem(PCG_PROBLEMS[tag])
    z = load_golden("pcg")
    t = f"{tag}_lm_{solver.replace('-', '_')}"
    tr, _, _ = O.lm_run(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points,
                        max_outer_iterations=10, max_order=2, solver=solver)
    its = tr.iterations
    assert len(its) == len(z[t + "_cost"])
    np.testing.assert_allclose([i.cost for i in its], z[t + "_cost"], rtol=1e-10)
    assert [i.inner for i in its][1:] == z[t + "_inner"].tolist()[1:]
    assert [i.order_m for i in its][1:] == z[t + "_order"].tolist()[1:]
    assert [i.accepted for i in its] == z[t + "_accepted"].tolist()
    np.testing.assert_allclose([i.lam for i in its], z[t + "_lam"], rtol=0)


# -- PoBA-32 (precision=32), pinned by tests/golden/p32.npz --------------------------------

@pytest.mark.parametrize("tag", ["c1", "mixed"])
def test_poba32_matches_reference(tag):
    p, _ = golden_problem(tag)
    z = load_golden("p32")
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points, precision=32)
    assert np.array_equal(lin.store.astype(np.float32).astype(np.float64), lin.store)
    for key in ("U0", "V0", "b_p", "b_l", "D_p", "D_l"):
        assert rel(getattr(lin, key), z[f"{tag}_{key}"]) < 1e-13, key
    s = O.OracleSystem(lin, 1e-4)
    assert rel(s.b_tilde(), z[f"{tag}_sys_b_tilde"]) < 1e-11
    for j in range(2):
        pre = f"{tag}_sys_solve{j}_"
        dp, order, conv = O.series_solve(s, float(z[pre + "eps"]), int(z[pre + "m"]))
        assert order == int(z[pre + "order"]) and conv == bool(z[pre + "converged"])
        assert rel(dp, z[pre + "delta_p"]) < 1e-10
        assert rel(O.back_sub(s, dp), z[pre + "delta_l"]) < 1e-10
    tr, _, _ = O.lm_run(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points,
                        max_outer_iterations=12, max_order=20, precision=32)
    np.testing.assert_allclose([i.cost for i in tr.iterations], z[f"{tag}_lm32_cost"], rtol=1e-10)
    assert [i.accepted for i in tr.iterations] == z[f"{tag}_lm32_accepted"].tolist()


# -- spectral diagnostics (reference spectral.py), pinned by tests/golden/spectral.npz ------

SPECTRAL = {"c1": "c1", "noisy": "noisy4x60", "mixed": "mixed"}


@pytest.mark.parametrize("tag", sorted(SPECTRAL))
def test_spectral_matches_reference(tag):
    p, _ = golden_problem(SPECTRAL[tag])
    z = load_golden("spectral")
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    for j in range(2):
        pre = f"{tag}_l{j}_"
        s = O.OracleSystem(lin, float(z[pre + "lam"]))
        val, it, conv = O.estimate_spectral_radius(s, tol=1e-4, max_iter=20000, seed=0)
        want = z[pre + "rho_loose"]
        assert abs(val - want[0]) <= 1e-10 * want[0] and it == int(want[1]) and conv == bool(want[2])
        rho, orders, bound, measured, un, bn = O.verify_error_bound(s, [0, 1, 2, 4, 8])
        assert abs(rho - float(z[pre + "rho_dense"])) <= 1e-9
        np.testing.assert_allclose(measured, z[pre + "measured"], rtol=1e-6)
        np.testing.assert_allclose(bound, z[pre + "bound"], rtol=1e-6)
        np.testing.assert_allclose([un, bn], z[pre + "norms"], rtol=1e-12)


# -- PoST clustering (reference clustering.py), pinned by tests/golden/post.npz -------------

POST = {"c1": "c1", "mixed": "mixed", "c2": "c2"}


@pytest.mark.parametrize("tag", sorted(POST))
def test_post_clustering_matches_reference(tag):
    p, _ = golden_problem(POST[tag])
    z = load_golden("post")
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points) if tag != "c2" else None
    for size in (1, 5, 16, 1000):
        pre = f"{tag}_s{size}_"
        a, n, sizes, cut = O.cluster_cameras(p.cam_indices, p.pt_indices, p.n_cameras, size)
        assert np.array_equal(a, z[pre + "assignment"]) and [n, cut] == z[pre + "meta"].tolist()
        assert np.array_equal(sizes, z[pre + "sizes"])
        if lin is None:
            continue
        for j, lam in enumerate([1e-4, 1.0]):
            for k, (eps, m) in enumerate([(0.01, 20), (1e-300, 6)]):
                q = pre + f"l{j}_e{k}_"
                dp, order, conv = O.solve_clustered(lin, lam, a, n, eps, m)
                assert [order, conv] == z[q + "order_conv"].tolist()
                assert rel(dp, z[q + "delta_p"]) < 1e-10


# ---- the C restatement of W / W^T used for configuration-scale parity -------------------

@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("threads", [1, 3])
def test_scale_oracle_matches_reference(name, threads):
    """oracle/poba_term.c (ScaleOracleSystem) reproduces the reference's golden
    b_tilde, series increments and back-substitutions, and the numpy oracle's
    W / W^T passes to a few ulps, for any thread count."""
    if O.term_library() is None:
        pytest.skip("oracle/lib/libpoba_oracle.so not built (make oracle)")
    p, z = golden_problem(name)
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    j = 0
    while f"lam{j}" in z:
        s = O.ScaleOracleSystem(lin, float(z[f"lam{j}"]), threads=threads)
        ref = O.OracleSystem(lin, float(z[f"lam{j}"]))
        rng = np.random.default_rng(j)
        vp, vl = rng.standard_normal(9 * p.n_cameras), rng.standard_normal(3 * p.n_points)
        assert rel(s.apply_wt(vp), ref.apply_wt(vp)) < 1e-14
        assert rel(s.apply_w(vl), ref.apply_w(vl)) < 1e-14
        assert rel(s.b_tilde(), z[f"sys{j}_b_tilde"]) < 1e-12
        i = 0
        while f"sys{j}_solve{i}_eps" in z:
            pre = f"sys{j}_solve{i}_"
            dp, order, conv = O.series_solve(s, float(z[pre + "eps"]), int(z[pre + "m"]))
            assert order == int(z[pre + "order"]) and conv == bool(z[pre + "converged"])
            assert rel(dp, z[pre + "delta_p"]) < 1e-11
            assert rel(O.back_sub(s, dp), z[pre + "delta_l"]) < 1e-11
            i += 1
        j += 1


def test_scale_oracle_at_medium_size():
    """C3 x 0.2 (~175k observations, hundreds of landmark runs per thread):
    C passes vs the numpy restatement."""
    if O.term_library() is None:
        pytest.skip("oracle/lib/libpoba_oracle.so not built (make oracle)")
    from paper_2204_12834_b200 import configs
    p = configs.make_config("c3", 0.2, seed=0)
    lin = O.linearize(p.cam_indices, p.pt_indices, p.pixels, p.camera_params, p.points)
    s, ref = O.ScaleOracleSystem(lin, 1e-4, threads=4), O.OracleSystem(lin, 1e-4)
    vp = np.random.default_rng(3).standard_normal(9 * p.n_cameras)
    assert rel(s.apply_w(s.apply_v_inv(s.apply_wt(vp))), ref.apply_w(ref.apply_v_inv(ref.apply_wt(vp)))) < 1e-13
