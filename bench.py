"""Benchmark: power-series Schur solve throughput on BASELINE.json configs[4] (C5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c5] [--scale 1.0]

A step is one power-series solve of the damped reduced camera system
(power_series_solve with the config's m = 32, epsilon = 0.01; b_tilde + up to m
terms, each term = W^T -> V^-1 -> W -> U^-1 over all observations) on the
synthetic C5 problem (13,700 cameras, 4.5M points, ~29M observations) at its
initial linearization, lambda = 1e-4.  `value` is series terms per second of
the whole job (inputs resident in HBM, device-timed with CUDA events on the
library stream, max over ranks); `e2e` is the same metric through the public
Python API with the state in pinned host memory and host<->device copies
inside the timed region (linearize + damp + series + back-substitution).
For N > 1 (torchrun) landmarks are sharded across ranks and every term ends
with one NCCL all-reduce of the 9*n_cam camera vector (strong scaling).

--impl reference times the reference's own CPU path: the unmodified reference
package shipped in baseline/_ref (installed by __graft_entry__.build()),
one full-size series term per step on one pinned core (the oracle port in
oracle/ stands in only if baseline/_ref is absent, and the line says so).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "power-series Schur solve iters/s"
UNIT = "iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def term_bytes(n_obs, n_lm, n_cam):
    """Algorithmic HBM bytes of one series term."""
    return 196 * n_obs + 48 * n_lm + 648 * n_cam


def kernel_bytes(n_obs, n_lm, n_cam):
    """Algorithmic bytes of one launch of the fused term kernel: J (192 B) + camera
    index (4 B) per observation, packed V^-1 (48 B) per landmark, the camera
    vector read (72 B) per camera."""
    return 196 * n_obs + 48 * n_lm + 72 * n_cam


def measured_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(problem, target_obs=1_500_000):
    """Spatially contiguous sub-problem (landmark-index prefix) of about target_obs observations."""
    from paper_2204_12834_b200.problem import Problem
    k = np.bincount(problem.pt_indices, minlength=problem.n_points)
    cum = np.cumsum(k)
    n_pts = int(np.searchsorted(cum, min(target_obs, cum[-1]))) + 1
    sel = problem.pt_indices < n_pts
    cams = np.unique(problem.cam_indices[sel])
    cmap = -np.ones(problem.n_cameras, dtype=np.int64)
    cmap[cams] = np.arange(len(cams))
    sub = Problem(problem.camera_params[cams], problem.points[:n_pts], cmap[problem.cam_indices[sel]],
                  problem.pt_indices[sel], problem.pixels[sel], name="sample")
    return sub


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def pin_one_core():
    """the reference runs on one pinned core with BLAS threads = 1."""
    cores = sorted(os.sched_getaffinity(0))
    os.sched_setaffinity(0, {cores[-1]})
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    return len(cores)


def reference_system(problem, lam):
    """The unmodified reference (``powerba`` shipped in baseline/_ref) assembles the
    damped system through its own public API; falls back to the oracle port
    (oracle/, the same algorithm restated) when the package is absent.
    Returns (system, power_series_solve, kind, setup_s)."""
    t0 = time.perf_counter()
    if os.path.isdir(os.path.join(REF_DIR, "powerba")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from powerba import blocks as rblocks
        from powerba.bal_io import BalProblem
        from powerba.power_series import power_series_solve
        bp = BalProblem(problem.camera_params, problem.points, problem.cam_indices, problem.pt_indices,
                        problem.pixels, name=getattr(problem, "name", ""))
        s = rblocks.assemble(bp, lam=lam)
        s.b_tilde()  # cached, as BASELINE.md section 3 prescribes
        return s, power_series_solve, "reference", time.perf_counter() - t0
    from oracle import poba_oracle as O
    lin = O.linearize(problem.cam_indices, problem.pt_indices, problem.pixels, problem.camera_params,
                      problem.points)
    s = O.OracleSystem(lin, lam)
    s.b_tilde()

    def solve(system, epsilon, max_order):
        return O.series_solve(system, epsilon, max_order)
    return s, solve, "port", time.perf_counter() - t0


def cpu_term_timer(problem, lam):
    """CPU baseline on a bounded sample: the reference's power_series_solve with
    max_order = 1 (U^-1 rhs + one term W^T, V^-1, W, U^-1) on a spatially
    contiguous 1.5M-observation prefix of the same problem, one pinned core;
    the per-observation rate is scaled to the full workload."""
    sub = cpu_sample(problem)
    n_host = pin_one_core()
    s, solve, kind, setup = reference_system(sub, lam)

    def one_term():
        t0 = time.perf_counter()
        solve(s, 1e-300, 1)
        return time.perf_counter() - t0

    desc = (f"{'reference powerba (baseline/_ref)' if kind == 'reference' else 'oracle port'} "
            f"power_series_solve(max_order=1) = one series term (+ U^-1 of the rhs) on a "
            f"{sub.n_observations}-obs / {sub.n_points}-landmark / {sub.n_cameras}-camera landmark-index prefix "
            f"of the workload, scaled per observation to {problem.n_observations} obs; 1 pinned core of "
            f"{n_host}, BLAS threads 1")
    return one_term, sub.n_observations, desc, kind


def run_reference(args):
    """--impl reference: the reference's own CPU path at the FULL workload size.

    The unmodified reference package (baseline/_ref) assembles the damped
    system of the bench config (its linearize + damp + cached b_tilde, untimed
    setup), then every step is one ``power_series_solve(system, 1e-300, 1)``
    = one full-size series term (plus one U^-1 of the right-hand side), timed
    with perf_counter on one pinned core.  Under
    torchrun only rank 0 runs."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2204_12834_b200 import configs
    problem = configs.make_config(args.config, args.scale, seed=0)  # all cores; not timed
    st = configs.LM_SETTINGS.get(args.config, configs.LmSettings())
    n_host = pin_one_core()
    s, solve, kind, setup = reference_system(problem, st.initial_lambda)
    for _ in range(args.warmup):
        solve(s, 1e-300, 1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        solve(s, 1e-300, 1)
        times.append(time.perf_counter() - t0)
    per_term = sum(times) / len(times)
    value = 1.0 / per_term
    desc = (f"{'reference powerba (baseline/_ref), unmodified' if kind == 'reference' else 'oracle port'}: "
            f"power_series_solve(system, 1e-300, max_order=1) per step = one series term (+ U^-1 of the rhs) "
            f"on the full {problem.n_observations}-obs problem; assemble + b_tilde setup {setup:.1f} s untimed; "
            f"1 pinned core of {n_host} host cores, BLAS threads 1")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per_term,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "n_observations": problem.n_observations,
                                            "n_cameras": problem.n_cameras, "n_points": problem.n_points,
                                            "lambda": st.initial_lambda},
            "setup_s": setup, "step_s": times,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch(args):
    """--gpus N (N > 1) without a torchrun environment: re-launch this script as
    N ranks under torch.distributed.run on 127.0.0.1 (rank 0 prints the line)."""
    import socket
    import torch
    n_vis = torch.cuda.device_count()
    if n_vis < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {n_vis} GPU(s) are visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus and args.gpus != 1:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        # communicator INFO lines (nranks, rings / NVLS) stay on stderr for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2204_12834_b200 import _lib, blocks, configs
    import paper_2204_12834_b200 as P

    problem = configs.make_config(args.config, args.scale, seed=0)
    st = configs.LM_SETTINGS.get(args.config, configs.LmSettings())
    lam, eps, m = st.initial_lambda, st.epsilon, st.max_order

    nccl_id = None
    if world > 1:
        obj = [_lib.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    dp = blocks.DeviceProblem(problem.cam_indices, problem.pt_indices, problem.pixels, problem.n_cameras,
                              problem.n_points, device=local, rank=rank, nranks=world, nccl_id=nccl_id)
    object.__setattr__(problem, "_poba_device", (blocks._signature(problem), blocks._snapshot(problem), dp))
    dev = dp.dev
    info = dev.info()

    # the system at the initial linearization (device resident)
    dev.set_points(problem.points)
    dev.linearize(problem.camera_params)
    dev.damp(lam)
    stream = torch.cuda.ExternalStream(dev.stream_ptr(), device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        dev.series_solve(eps, m)
    barrier()
    clocks = ClockSampler(local)
    l0 = dev.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    terms = 0
    e0.record(stream)
    for _ in range(args.steps):
        _, order, _, _ = dev.series_solve(eps, m)
        terms += order
    e1.record(stream)
    e1.synchronize()
    barrier()
    clock_info = clocks.stop()
    launches = dev.launch_count() - l0
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = terms / (ms / 1e3)
    ms_per_step = ms / args.steps

    # dominant kernel: the fused term kernel, timed alone with CUDA events in the library
    ms_term, ms_kernel, launches_per_term = dev.time_terms(20)
    n_obs_l, n_lm_l = info["n_obs_local"], info["lm_hi"] - info["lm_lo"]
    peak, peak_kind = measured_peak()
    kb = kernel_bytes(n_obs_l, n_lm_l, problem.n_cameras)
    achieved = kb / (ms_kernel / 1e3) / 1e9
    traffic = None
    prof = os.path.join(REPO, "profiles", f"term_traffic_{args.config}.json")
    if os.path.exists(prof) and args.scale == 1.0 and world == 1:
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    tb_total = term_bytes(problem.n_observations, problem.n_points, problem.n_cameras)

    # end to end through the public API, host state in pinned memory
    e2e = None
    if not args.no_e2e:
        cams_h = torch.from_numpy(problem.camera_params).pin_memory().numpy()
        pts_h = torch.from_numpy(problem.points).pin_memory().numpy()

        class State:
            camera_params = cams_h
            points = pts_h
        for _ in range(2):
            s = P.assemble(problem, State, lam=lam)
            r = P.power_series_solve(s, eps, m)
            P.back_substitute(s, r.delta_p)
        barrier()
        e_terms = 0
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s = P.assemble(problem, State, lam=lam)
            r = P.power_series_solve(s, eps, m)
            P.back_substitute(s, r.delta_p)
            e_terms += r.order_used
        torch.cuda.synchronize()
        e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t.item())
        n_c, n_l = problem.n_cameras, problem.n_points
        e2e = {"value": e_terms / e_s, "unit": UNIT, "ms_per_step": 1e3 * e_s / args.steps,
               "h2d_bytes_per_step": (9 * n_c + 3 * n_l + 9 * n_c) * 8,
               "d2h_bytes_per_step": (9 * n_c + 3 * n_l) * 8,
               "path": "blocks.assemble (linearize+damp) -> power_series_solve -> back_substitute"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        one_term, n_s, desc, kind = cpu_term_timer(problem, lam)
        one_term()
        ts = [one_term() for _ in range(3)]
        per_full = (sum(ts) / len(ts)) * problem.n_observations / n_s
        cpu = {"value": 1.0 / per_full, "unit": UNIT, "cores": 1, "kind": kind, "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator for BASELINE.json configs; no BAL data offline)",
            "config": {"workload": args.config, "scale": args.scale, "n_cameras": problem.n_cameras,
                       "n_points": problem.n_points, "n_observations": problem.n_observations,
                       "max_order": m, "epsilon": eps, "lambda": lam, "terms_per_step": terms / args.steps,
                       "l2": f"inputs larger than L2 (store {info['device_bytes'] / 1e9:.1f} GB per GPU)",
                       "parallelism": f"landmark-sharded x{world}, NCCL all-reduce per term" if world > 1
                       else "single GPU"},
            "obs_per_s": value * problem.n_observations,
            "hbm_gbs_term": tb_total * value / 1e9 / max(world, 1),
            "roofline": {"bound": "hbm", "kernel": "k_term (fused W^T V^-1 W series term)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_kind": peak_kind, "traffic": traffic, "bytes_per_launch": kb,
                         "ms_per_launch": ms_kernel, "ms_per_term_all_kernels": ms_term,
                         "launches_per_term": launches_per_term},
            "e2e": e2e, "gpu_launches": launches, "clocks": clock_info, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main() or 0)
