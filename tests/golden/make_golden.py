"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

It imports the reference package ``powerba`` (read-only source tree; bytecode
writing disabled) and records, for a handful of small problems, the outputs of
the reference's own hot-path functions: ``blocks._sorted_observation_order``,
``blocks.linearize`` / ``assemble_from_observations``, ``Linearization.damp``,
``DampedSystem.b_tilde``, ``power_series_solve``, ``back_substitute``,
``lm.residual_cost`` and ``lm.run`` (reference ``pkg/src/powerba``).  The GPU
box never sees /root/reference; tests only read the .npz files written here.
"""
from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))

import numpy as np  # noqa: E402
from powerba import bal_io, blocks, lm, solvers, synthetic  # noqa: E402
from powerba.power_series import back_substitute, power_series_solve  # noqa: E402

import helpers  # noqa: E402  (the reference's own test oracles: random_block_system)


def problem_arrays(p):
    return dict(camera_params=p.camera_params, points=p.points, cam_indices=p.cam_indices,
                pt_indices=p.pt_indices, pixels=p.pixels)


def lin_outputs(lin, prefix="", store=True):
    st = lin.store
    out = {
        prefix + "cam_sorted": st.cam_sorted, prefix + "pt_sorted": st.pt_sorted,
        prefix + "group_k": np.array([g.k for g in st.groups]),
        prefix + "group_start": np.array([g.obs_start for g in st.groups]),
        prefix + "group_n": np.array([g.n for g in st.groups]),
        prefix + "U0": lin.U0, prefix + "V0": lin.V0, prefix + "b_p": lin.b_p,
        prefix + "b_l": lin.b_l, prefix + "D_p": lin.D_p, prefix + "D_l": lin.D_l,
        prefix + "n_invalid": np.array(lin.n_invalid),
    }
    if store:
        out[prefix + "storage"] = st.storage_obs
    return out


def system_outputs(sys_, tag, solves):
    out = {f"{tag}_U_inv": sys_.U_inv, f"{tag}_V_inv": sys_.V_inv,
           f"{tag}_b_tilde": sys_.b_tilde()}
    for j, (eps, m) in enumerate(solves):
        r = power_series_solve(sys_, epsilon=eps, max_order=m)
        out[f"{tag}_solve{j}_eps"] = np.array(eps)
        out[f"{tag}_solve{j}_m"] = np.array(m)
        out[f"{tag}_solve{j}_delta_p"] = r.delta_p
        out[f"{tag}_solve{j}_order"] = np.array(r.order_used)
        out[f"{tag}_solve{j}_converged"] = np.array(r.converged)
        out[f"{tag}_solve{j}_delta_l"] = back_substitute(sys_, r.delta_p)
    return out


def trace_outputs(trace, tag):
    its = trace.iterations
    return {f"{tag}_cost": np.array([i.cost for i in its]),
            f"{tag}_lam": np.array([i.lam for i in its]),
            f"{tag}_order": np.array([i.order_m for i in its]),
            f"{tag}_accepted": np.array([i.accepted for i in its]),
            f"{tag}_n_invalid": np.array([i.n_invalid for i in its]),
            f"{tag}_peak_bytes": np.array([i.peak_bytes for i in its]),
            f"{tag}_converged": np.array(trace.converged)}


def bundle(name, p, *, lams, solves, lm_cfgs, store=True, save_inputs=True):
    out = {"name": np.array(name)}
    if save_inputs:
        out.update(problem_arrays(p))
    from paper_2204_12834_b200.problem import Problem
    out["fingerprint"] = np.array(Problem(**problem_arrays(p)).fingerprint())
    cs, ps, order = blocks._sorted_observation_order(p.cam_indices, p.pt_indices, p.n_points)
    out["order"] = order
    lin = blocks.linearize(p)
    out.update(lin_outputs(lin, store=store))
    out["cost0"] = np.array(lm.residual_cost(p, lm.BaState.from_problem(p)))
    for j, lam in enumerate(lams):
        out[f"lam{j}"] = np.array(lam)
        out.update(system_outputs(lin.damp(lam), f"sys{j}", solves))
    for tag, cfg in lm_cfgs.items():
        tr = lm.run(p, cfg)
        out.update(trace_outputs(tr, tag))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"wrote {name}.npz ({p.n_cameras} cams, {p.n_points} pts, {p.n_observations} obs)")


def explicit_bundle():
    """Systems built by assemble_from_observations (the reference's test seam)."""
    out = {}
    for j, (seed, lam) in enumerate([(0, 1e-4), (1, 1e-2), (2, 1.0), (4, 1e-2)]):
        rng = np.random.default_rng(seed)
        n_cam = int(rng.integers(2, 11))
        n_pt = int(rng.integers(8, 51))
        # same recipe as helpers.random_block_system (tests/helpers.py:200-233)
        cam_idx = list(np.repeat(np.arange(n_cam), n_pt))
        pt_idx = list(np.tile(np.arange(n_pt), n_cam))
        nv = len(cam_idx)
        jp = [rng.normal(size=(nv, 2, 9))]
        jl = [rng.normal(size=(nv, 2, 3))]
        res = [rng.normal(size=(nv, 2))]
        for c in range(n_cam):
            cam_idx.extend([c] * 5)
            pt_idx.extend(int(rng.integers(n_pt)) for _ in range(5))
            jp.append(3.0 * rng.normal(size=(5, 2, 9)))
            jl.append(np.zeros((5, 2, 3)))
            res.append(rng.normal(size=(5, 2)))
        cam_idx = np.array(cam_idx)
        pt_idx = np.array(pt_idx)
        jp, jl, res = np.concatenate(jp), np.concatenate(jl), np.concatenate(res)
        # duplicates (anchor rows repeat a visible pair) are allowed by this seam
        lin = blocks.assemble_from_observations(cam_idx, pt_idx, jp, jl, res, n_cam, n_pt)
        sys_ = lin.damp(lam)
        ref_sys = helpers.random_block_system(seed, lam=lam)
        assert np.array_equal(ref_sys.b_tilde(), sys_.b_tilde())
        pre = f"e{j}_"
        out.update({pre + "cam_idx": cam_idx, pre + "pt_idx": pt_idx, pre + "jp": jp,
                    pre + "jl": jl, pre + "res": res, pre + "n_cam": np.array(n_cam),
                    pre + "n_pt": np.array(n_pt), pre + "lam": np.array(lam)})
        out.update(lin_outputs(lin, pre, store=False))
        out.update(system_outputs(sys_, pre + "sys", [(1e-14, 200), (1e-300, 6), (0.01, 20)]))
    # decoupled system: J_l = 0 (tests/test_power_series.py:82-94)
    rng = np.random.default_rng(3)
    jp = rng.normal(size=(6, 2, 9))
    jl = np.zeros((6, 2, 3))
    res = rng.normal(size=(6, 2))
    ci, pi = np.array([0, 0, 0, 1, 1, 1]), np.array([0, 1, 2, 0, 1, 2])
    lin = blocks.assemble_from_observations(ci, pi, jp, jl, res, 2, 3)
    sys_ = lin.damp(1e-2)
    r = power_series_solve(sys_, epsilon=1e-12)
    out.update({"dec_jp": jp, "dec_jl": jl, "dec_res": res, "dec_cam_idx": ci, "dec_pt_idx": pi,
                "dec_delta_p": r.delta_p, "dec_order": np.array(r.order_used),
                "dec_u_inv_minus_bt": sys_.apply_u_inv(-sys_.b_tilde())})
    np.savez_compressed(os.path.join(HERE, "explicit.npz"), **out)
    print("wrote explicit.npz")


def pcg_bundle():
    """Reference PCG baselines (solvers.py:30-118) on the c1 and noisy4x60 problems."""
    from paper_2204_12834_b200 import configs
    out = {}
    probs = {"c1": configs.make_config("c1"),
             "noisy": bal_io.perturb(synthetic.make_random_problem(4, 60, seed=5, pixel_noise=1.0), 0.01, seed=0)}
    for tag, p in probs.items():
        out[f"{tag}_fingerprint"] = np.array(
            __import__("paper_2204_12834_b200.problem", fromlist=["Problem"]).Problem(**problem_arrays(p)).fingerprint())
        lin = blocks.linearize(p)
        for j, lam in enumerate([1e-4, 1.0]):
            sys_ = lin.damp(lam)
            pre = f"{tag}_l{j}_"
            out[pre + "lam"] = np.array(lam)
            out[pre + "schur_diag"] = solvers.schur_diagonal_blocks(sys_)
            rels = []
            rep = solvers.pcg_schur_jacobi(sys_, 1e-6, 500, callback=lambda it, x, rel: rels.append(rel))
            out[pre + "jac_delta_p"], out[pre + "jac_iters"] = rep.delta_p, np.array(rep.iterations)
            out[pre + "jac_rel"], out[pre + "jac_conv"] = np.array(rep.final_relative_residual), np.array(rep.converged)
            out[pre + "jac_rels"] = np.array(rels)
            for m in (0, 2):
                rep = solvers.pcg_power_series_preconditioner(sys_, m, 1e-6, 500)
                out[pre + f"pow{m}_delta_p"], out[pre + f"pow{m}_iters"] = rep.delta_p, np.array(rep.iterations)
                out[pre + f"pow{m}_rel"] = np.array(rep.final_relative_residual)
            rep = solvers.pcg_schur_jacobi(sys_, 1e-3, 3)
            out[pre + "jac3_delta_p"], out[pre + "jac3_iters"] = rep.delta_p, np.array(rep.iterations)
            out[pre + "jac3_conv"] = np.array(rep.converged)
        for solver in ("pcg", "pcg-power"):
            cfg = lm.LmConfig(solver=solver, max_outer_iterations=10, max_order=2)
            tr = lm.run(p, cfg)
            its = tr.iterations
            t = f"{tag}_lm_{solver.replace('-', '_')}"
            out[t + "_cost"] = np.array([i.cost for i in its])
            out[t + "_lam"] = np.array([i.lam for i in its])
            out[t + "_inner"] = np.array([i.inner_iterations for i in its])
            out[t + "_order"] = np.array([i.order_m for i in its])
            out[t + "_accepted"] = np.array([i.accepted for i in its])
    np.savez_compressed(os.path.join(HERE, "pcg.npz"), **out)
    print("wrote pcg.npz")


def mixed_bundle():
    """Track lengths 1 .. 72 (single-observation points, packed short tracks, long tracks)."""
    from paper_2204_12834_b200 import configs
    mixed = configs.make_mixed_tracks()
    p = bal_io.BalProblem(mixed.camera_params, mixed.points, mixed.cam_indices, mixed.pt_indices, mixed.pixels)
    bundle("mixed", p, lams=[1e-4, 1.0], solves=[(0.01, 20), (1e-300, 12)],
           lm_cfgs={"lm_mixed": lm.LmConfig(solver="poba", max_outer_iterations=15, max_order=20)})


def p32_bundle():
    """PoBA-32 (precision=32: float32 block storage, float64 reductions) on c1 and mixed."""
    from paper_2204_12834_b200 import configs
    out = {}
    mixed = configs.make_mixed_tracks()
    probs = {"c1": configs.make_config("c1"),
             "mixed": bal_io.BalProblem(mixed.camera_params, mixed.points, mixed.cam_indices, mixed.pt_indices,
                                        mixed.pixels)}
    for tag, p in probs.items():
        lin = blocks.linearize(p, precision=32)
        assert lin.store.storage_obs.dtype == np.float32
        out.update(lin_outputs(lin, f"{tag}_"))
        out.update(system_outputs(lin.damp(1e-4), f"{tag}_sys", [(0.01, 20), (1e-300, 12)]))
        out.update(trace_outputs(lm.run(p, lm.LmConfig(solver="poba", precision=32, max_outer_iterations=12,
                                                       max_order=20)), f"{tag}_lm32"))
    np.savez_compressed(os.path.join(HERE, "p32.npz"), **out)
    print("wrote p32.npz")


BAL_CASES = {
    # name: text (the reference's own parser decides what each one means)
    "minimal": "1 1 1\n0 0 1.5 -2.25\n" + " ".join(["0.1"] * 9) + "\n1 2 3\n",
    "layout_free": "1 1\n1 0 0\n1.5 -2.25 " + " ".join(["0.1"] * 9) + " 1\n2\n\n3",
    "tabs_crlf": "1\t1\t1\r\n0 0 1.5 -2.25\r\n" + " ".join(["0.1"] * 9) + "\r\n1 2 3\r\n",
    "numbers": "1 2 2\n0 0 +1_0.5e-1_0 .5\n0_0 1 1 2\n" + " ".join(["0.1"] * 9) + "\n1 2 3 4 5 6\n",
    "number_forms": "2 2 2\n0 0 1e400 -inf\n1 1 NaN 5.\n" + " ".join(["1E-320"] * 9) + " "
                    + " ".join(["-0.0"] * 9) + "\n1 2 3 4 5 6\n",
    "plus_index": "1 1 1\n+0 00 1 2\n" + " ".join(["0.1"] * 9) + "\n1 2 3\n",
    "prune": "3 3 2\n0 0 1 2\n2 2 3 4\n" + " ".join(["0.1"] * 27) + "\n" + " ".join(["1"] * 9) + "\n",
    "point_range": "1 1 1\n0 1 1 2\n",
    "camera_range": "1 1 1\n-1 0 1 2\n",
    "duplicate": "1 1 2\n0 0 1 2\n0 0 3 4\n",
    "truncated_obs": "1 1 2\n0 0 1 2\n0\n",
    "truncated_cam": "1 1 1\n0 0 1 2\n0.1 0.2\n\n\n",
    "truncated_pt": "1 1 1\n0 0 1 2\n" + " ".join(["0.1"] * 9) + "\n1 2",
    "non_numeric": "1 1 1\n0 0 abc 2\n",
    "hex_float": "1 1 1\n0 0 0x1p3 2\n",
    "underscore_bad": "1 1 1\n0 0 1__0 2\n",
    "non_integer_index": "1 1 1\n0.0 0 1 2\n",
    "quote_token": "1 1 1\n0 0 it's 2\n",
    "trailing": "1 1 1\n0 0 1 2\n" + " ".join(["0.1"] * 9) + "\n1 2 3\n\n4\n",
    "zero_count": "0 1 1\n",
    "negative_count": "1 -2 1\n",
    "empty": "",
    "header_only": "1 1 1\n",
    "bad_header": "x 1 1\n",
    "huge_index": "1 1 1\n123456789012345678901234567890 0 1 2\n",
}


def bal_bundle():
    """The reference's own parse_bal on a corpus of BAL texts: arrays or error messages."""
    import io
    out = {}
    for name, text in BAL_CASES.items():
        out[f"{name}_text"] = np.frombuffer(text.encode(), dtype=np.uint8)
        try:
            p = bal_io.parse_bal(io.StringIO(text))
            out[f"{name}_ok"] = np.array(True)
            for k in ("camera_params", "points", "cam_indices", "pt_indices", "pixels"):
                out[f"{name}_{k}"] = getattr(p, k)
            out[f"{name}_pruned"] = np.array([p.n_pruned_cameras, p.n_pruned_points])
        except Exception as e:  # noqa: BLE001 -- record exactly what the reference raises
            out[f"{name}_ok"] = np.array(False)
            out[f"{name}_error"] = np.array(f"{type(e).__name__}: {e}")
    rig = synthetic.make_rig_problem(pixel_noise=1.0)
    text = bal_io.serialize_bal(bal_io.perturb(rig, 0.01, seed=0))
    out["rig_text"] = np.frombuffer(text.encode(), dtype=np.uint8)
    p = bal_io.parse_bal(io.StringIO(text))
    for k in ("camera_params", "points", "cam_indices", "pt_indices", "pixels"):
        out[f"rig_{k}"] = getattr(p, k)
    np.savez_compressed(os.path.join(HERE, "bal.npz"), **out)
    print("wrote bal.npz")


def spectral_bundle():
    """The reference's spectral diagnostics (spectral.py:54-143) on small systems."""
    from paper_2204_12834_b200 import configs
    from powerba import spectral
    out = {}
    mixed = configs.make_mixed_tracks()
    probs = {"c1": configs.make_config("c1"),
             "noisy": bal_io.perturb(synthetic.make_random_problem(4, 60, seed=5, pixel_noise=1.0), 0.01, seed=0),
             "mixed": bal_io.BalProblem(mixed.camera_params, mixed.points, mixed.cam_indices, mixed.pt_indices,
                                        mixed.pixels)}
    for tag, p in probs.items():
        lin = blocks.linearize(p)
        for j, lam in enumerate([1e-4, 1.0]):
            sys_ = lin.damp(lam)
            pre = f"{tag}_l{j}_"
            out[pre + "lam"] = np.array(lam)
            for tol_tag, tol in (("tight", 1e-9), ("loose", 1e-4)):
                est = spectral.estimate_spectral_radius(sys_, tol=tol, max_iter=20000, seed=0)
                out[pre + f"rho_{tol_tag}"] = np.array([est.value, est.iterations, est.converged])
            rep = spectral.verify_error_bound(sys_, [0, 1, 2, 4, 8])
            out[pre + "rho_dense"] = np.array(rep.rho)
            out[pre + "bound"], out[pre + "measured"] = rep.bound, rep.measured_error
            out[pre + "norms"] = np.array([rep.u_inv_norm, rep.b_tilde_norm])
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), **out)
    print("wrote spectral.npz")


def post_bundle():
    """The reference's PoST pieces (clustering.py): covisibility clusters, clustered solves, LM(post)."""
    from paper_2204_12834_b200 import configs
    from powerba import clustering
    out = {}
    mixed = configs.make_mixed_tracks()
    probs = {"c1": configs.make_config("c1"),
             "mixed": bal_io.BalProblem(mixed.camera_params, mixed.points, mixed.cam_indices, mixed.pt_indices,
                                        mixed.pixels),
             "c2": configs.make_config("c2")}
    for tag, p in probs.items():
        lin = blocks.linearize(p)
        for size in (1, 5, 16, 1000):
            part = clustering.cluster_cameras(p, size)
            pre = f"{tag}_s{size}_"
            out[pre + "assignment"] = part.assignment
            out[pre + "meta"] = np.array([part.n_clusters, part.cut_observations])
            out[pre + "sizes"] = part.sizes
            if tag != "c2":
                for j, lam in enumerate([1e-4, 1.0]):
                    sys_ = lin.damp(lam)
                    for k, (eps, m) in enumerate([(0.01, 20), (1e-300, 6)]):
                        r = clustering.solve_clustered(sys_, part, eps, m)
                        q = pre + f"l{j}_e{k}_"
                        out[q + "delta_p"] = r.delta_p
                        out[q + "order_conv"] = np.array([r.order_used, r.converged])
        if tag != "c2":
            tr = lm.run(p, lm.LmConfig(solver="post", max_cluster_size=5, max_outer_iterations=10, max_order=20))
            out.update(trace_outputs(tr, f"{tag}_lm_post"))
    np.savez_compressed(os.path.join(HERE, "post.npz"), **out)
    print("wrote post.npz")


def direct_bundle():
    """The reference's dense_direct (solvers.py:136-151) and lm.run(solver="direct")."""
    from paper_2204_12834_b200 import configs
    out = {}
    probs = {"c1": configs.make_config("c1"),
             "noisy": bal_io.perturb(synthetic.make_random_problem(4, 60, seed=5, pixel_noise=1.0), 0.01, seed=0)}
    for tag, p in probs.items():
        lin = blocks.linearize(p)
        for j, lam in enumerate([1e-4, 1.0]):
            out[f"{tag}_l{j}_delta_p"] = solvers.dense_direct(lin.damp(lam))
        out.update(trace_outputs(lm.run(p, lm.LmConfig(solver="direct", max_outer_iterations=10)), f"{tag}_lm_direct"))
    np.savez_compressed(os.path.join(HERE, "direct.npz"), **out)
    print("wrote direct.npz")


def main():
    if len(sys.argv) > 2 and sys.argv[2] == "direct":
        return direct_bundle()
    if len(sys.argv) > 2 and sys.argv[2] == "post":
        return post_bundle()
    if len(sys.argv) > 2 and sys.argv[2] == "spectral":
        return spectral_bundle()
    if len(sys.argv) > 2 and sys.argv[2] == "bal":
        return bal_bundle()
    if len(sys.argv) > 2 and sys.argv[2] == "p32":
        return p32_bundle()
    if len(sys.argv) > 2 and sys.argv[2] == "pcg":
        return pcg_bundle()
    if len(sys.argv) > 2 and sys.argv[2] == "mixed":
        return mixed_bundle()
    from paper_2204_12834_b200 import configs
    oracle = bal_io.perturb(synthetic.make_random_problem(3, 5, seed=1), 0.01, seed=0)
    bundle("rand3x5", oracle, lams=[1e-4, 1.0],
           solves=[(1e-12, 3), (1e-14, 50), (0.01, 20), (1e-300, 10)],
           lm_cfgs={"lm_poba": lm.LmConfig(solver="poba")})
    noisy = bal_io.perturb(synthetic.make_random_problem(4, 60, seed=5, pixel_noise=1.0), 0.01, seed=0)
    bundle("noisy4x60", noisy, lams=[1e-4, 1e-2],
           solves=[(0.01, 20), (1e-300, 12)],
           lm_cfgs={"lm_poba": lm.LmConfig(solver="poba")})
    rig = synthetic.make_rig_problem(pixel_noise=1.0)
    bundle("rig49", rig, lams=[1e-4], solves=[(0.01, 20), (1e-300, 32)],
           lm_cfgs={"lm_poba": lm.LmConfig(solver="poba", max_outer_iterations=50)}, store=False)
    c1 = configs.make_config("c1")
    bundle("c1", c1, lams=[1e-4], solves=[(0.01, 32), (1e-300, 32)],
           lm_cfgs={"lm_c1": lm.LmConfig(solver="poba", max_outer_iterations=10, max_order=32)},
           store=False)
    c2 = configs.make_config("c2")
    bundle("c2", c2, lams=[1e-4], solves=[(1e-6, 32)],
           lm_cfgs={"lm_c2": lm.LmConfig(solver="poba", max_outer_iterations=20, max_order=32,
                                         epsilon=1e-6)},
           store=False, save_inputs=False)
    explicit_bundle()
    pcg_bundle()
    mixed_bundle()
    p32_bundle()
    bal_bundle()
    spectral_bundle()
    post_bundle()
    direct_bundle()


if __name__ == "__main__":
    main()
