#!/usr/bin/env python
"""Benchmark of the hot path: block-preconditioned GMRES on the mixed-VEM
saddle-point system (BASELINE.json metric: time-to-solution & GMRES iters/s at
1 B200; SpMV / preconditioner HBM GB/s vs peak).

Workload: C5 (the largest single-GPU config of BASELINE.json: 96^3 cubes with ~50%
pairs, k = 1, anisotropic K with jumps, 14.0M DOFs) with the regularised block
preconditioner in its M-aware form (precond kind 5, R24).  One step = one
GMRES iteration (preconditioner apply + saddle SpMV + batched CGS): a C5 solve takes
minutes, so the K timed steps are the first K Arnoldi steps of solves from x0 = 0 (upload
and S_D build happen once, before timing: setup_ms).  value = GMRES iterations / s over
the K timed steps, all ranks; the time to solution of one complete solve to rtol 1e-10
is measured after the timed region (full_solve) with the per-kernel HBM rates, and C3
(round 1's headline) is timed as whole solves in `secondary`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Multi-GPU: "replicas only" — every rank solves its own copy of
the system; no collective on the data path.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution & GMRES iters/s at 1 B200; SpMV/precond HBM GB/s vs peak"
UNIT = "GMRES it/s"
ORACLE_ITS = os.path.join(ROOT, "profiles", "oracle_iterations.json")


def oracle_iterations(name, kind):
    """GMRES iterations the oracle itself needs for this workload (full-length CPU
    solve written by tools/oracle_iterations.py, oracle/ only); None if not recorded."""
    try:
        return int(json.load(open(ORACLE_ITS))[name][str(kind)]["iterations"])
    except Exception:
        return None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--precond", type=int, default=0, help="0 = the config's first preconditioner")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variant", action="store_true", help="skip the Block-Schur-AMG variant solve")
    ap.add_argument("--cpu-sample-its", type=int, default=6)
    ap.add_argument("--per-launch", action="store_true",
                    help="time every launch with events in the timed region (no graphs; ~10%% overhead)")
    ap.add_argument("--l2-persist", type=int, default=1)
    ap.add_argument("--reorth", type=int, default=-1, help="-1 auto (CGS1 for GMRES, CGS2 for FGMRES), 1 CGS2, 0 CGS1")
    return ap.parse_args()


def ncu_traffic(kclass):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel class
    from the committed `ncu --set full` capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(kclass)
        return None if e is None else e["bytes_per_launch"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and not s[2 + i].startswith("Not")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(self.samples)}


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, 0
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = "nccl" if args.impl == "ours" else "gloo"
    if backend == "nccl":
        import torch
        torch.cuda.set_device(local)
    dist.init_process_group(backend)
    return rank, ws, local


def headline_kind(cfg, system, args):
    """The approximate-Schur preconditioner of the config.  For
    n_p = 1 (C1, C3) its B_2 solve is the aggregation V-cycle on S_D (kind 3,
    DESIGN.md R22: the closer stand-in for the paper's exact MUMPS solve); the
    fixed-sweep Chebyshev-Jacobi form (kind 1) is timed beside it as `variant`."""
    if args.precond:
        return args.precond
    k = cfg.precs[0]
    if k == 1 and system.layout.n_p_dof == 1:
        return 3
    if cfg.name.startswith("C5"):
        return 5   # the regularised preconditioner with the M-aware velocity block (R24): kind 2 stagnates on C5
    return k


def reduce_over_ranks(ms: float, its: float, device="cpu"):
    """Replicas-only aggregation: the step time is the MAX over
    ranks, the work is the SUM of all ranks' GMRES iterations."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), float(its)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    w = torch.tensor([float(its)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t[0]), float(w[0])


def _cores():
    try:
        from threadpoolctl import threadpool_info
        return int(max([i.get("num_threads", 1) for i in threadpool_info()] + [1]))
    except Exception:
        return 1


def nested_counts(name):
    """K-PCG and inner-PCG steps per outer iteration of the kind-5 solve of `name`, from the
    last recorded full GPU solve (profiles/nested_counts.json, written by bench.py itself);
    the oracle reproduces these counts at reduced size (tests/test_gpu_blockreg_m.py)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "nested_counts.json")))[name]
    except Exception:
        return None


def cpu_baseline_nested(system, cfg, eps, counts, k_steps=1):
    """Kind 5 (PCG on K inside FGMRES): one outer iteration of the oracle on full C5 takes about
    20 minutes, so the bounded sample is `k_steps` steps of the PCG on K of the first non-trivial
    preconditioner apply (each: K p, the Woodbury block with its inner MG-PCG to k_inner_rtol,
    dots and updates), and GMRES it/s is EXTRAPOLATED as 1 / (K steps per outer iteration x
    seconds per K step + one saddle SpMV), with the K-steps-per-iteration count of the full GPU
    solve of the same system."""
    import numpy as np
    from oracle import solver as O
    t0 = time.perf_counter()
    P = O.Preconditioner(O.PRECOND_BLOCK_REG_M, system.M, system.B, eps=eps, block=system.layout.n_p_dof,
                         k_maxit=k_steps, k_rtol=1e-30)
    t1 = time.perf_counter()
    # second Krylov vector of the solve: v_1 ~ A P^-1 v_0 with v_0 = rhs / ||rhs|| (v_0 has no velocity part)
    z0 = P.apply(system.rhs / np.linalg.norm(system.rhs))
    w = O.spmv_saddle(system.M, system.B, z0)
    w /= np.linalg.norm(w)
    t2 = time.perf_counter()
    P.inner_iterations = 0
    P.k_iterations = 0
    P.apply(w)
    t3 = time.perf_counter()
    O.spmv_saddle(system.M, system.B, w)
    t4 = time.perf_counter()
    # one K step = (P.k_iterations steps + the initial Woodbury apply) / (k_steps + 1) applies
    per_k = (t3 - t2) / (P.k_iterations + 1)
    kpo = counts["k_per_outer"] if counts else None
    itps = 1.0 / (kpo * per_k + (t4 - t3)) if kpo else None
    return {"value": itps, "unit": UNIT, "cores": _cores(), "kind": "oracle", "extrapolated": True,
            "seconds_per_K_step": per_k, "K_steps_per_outer_iteration": kpo,
            "inner_steps_in_sample": int(P.inner_iterations),
            "sample": f"{P.k_iterations} step(s) of the PCG on K = M + B^T (eps W)^-1 B plus its initial Woodbury apply "
                      f"on the second Krylov vector of {cfg.name} (precond 5): {t3 - t2:.1f} s, {P.inner_iterations} inner "
                      f"MG-PCG steps (+{t1 - t0:.1f} s preconditioner setup, untimed); GMRES it/s EXTRAPOLATED with "
                      f"{kpo} K steps per outer iteration (full GPU solve of the same system, profiles/nested_counts.json)",
            "setup_s": t1 - t0}


def cpu_baseline(system, cfg, kind, eps, its):
    """The oracle as it stands on a bounded sample: `its` GMRES iterations of the
    same system on the host cores (value in GMRES it/s)."""
    from oracle import solver as O
    if kind == O.PRECOND_BLOCK_REG_M:
        return cpu_baseline_nested(system, cfg, eps, nested_counts(cfg.name))
    t0 = time.perf_counter()
    P = O.Preconditioner(kind, system.M, system.B, eps=eps, block=system.layout.n_p_dof)
    t1 = time.perf_counter()
    res = O.gmres(lambda x: O.spmv_saddle(system.M, system.B, x), P.apply, system.rhs, 1e-10, cfg.restart, its,
                  P.flexible, 1 if P.flexible else 0)
    t2 = time.perf_counter()
    itps = res.iterations / (t2 - t1)
    full = oracle_iterations(cfg.name, kind)
    return {"value": itps, "unit": UNIT, "cores": _cores(), "kind": "oracle", "extrapolated": False,
            "iterations_per_solve": full, "solves_per_s_extrapolated": (itps / full) if full else None,
            "sample": f"{res.iterations} GMRES iterations of {cfg.name} (precond {kind}) from x0=0, "
                      f"{t2 - t1:.1f} s (+{t1 - t0:.1f} s preconditioner setup, untimed)",
            "setup_s": t1 - t0}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (rank 0 only).  One step = one bounded
    sample (cpu_baseline); value = the mean GMRES it/s over the K samples; ms_per_step = the
    wall time of one sample (NOT of one GMRES iteration: see `sample`)."""
    rank, ws, _ = dist_init(args)
    if rank != 0:
        return
    from vemgen.configs import CONFIGS, eps_for
    cfg = CONFIGS[args.config]
    s = cfg.build()
    kind = headline_kind(cfg, s, args)   # the same preconditioner as our arm
    eps = eps_for(s)
    nested = kind == 5
    # kind 5: every sample costs ~25 s of oracle work, so the K + W samples are taken once
    # and the timing repeated on cached operators would be meaningless: one sample per step,
    # capped so that the run ends within a few minutes
    steps = min(args.steps, 4) if nested else args.steps
    warm = min(args.warmup, 1) if nested else args.warmup
    vals = []
    for _ in range(warm):
        cpu_baseline(s, cfg, kind, eps, 1)
    t0 = time.perf_counter()
    last = None
    for _ in range(steps):
        last = cpu_baseline(s, cfg, kind, eps, args.cpu_sample_its)
        vals.append(last["value"])
    dt = time.perf_counter() - t0
    value = sum(vals) / len(vals) if all(v is not None for v in vals) else None
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": (1e3 / value) if value else None,
            "samples_taken": steps, "warmup_samples_taken": warm, "ms_per_sample": 1e3 * dt / steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded vemgen assembly)",
            "config": {"workload": f"{cfg.name}: {cfg.describe}", "rtol": cfg.rtol, "restart": cfg.restart,
                       "precond": kind, "n_dofs": s.n,
                       "step": "one bounded oracle sample converted to GMRES it/s; ms_per_step = 1000 / value "
                               "(the time of one GMRES iteration at the sampled rate)"},
            "cpu_baseline": {k: last[k] for k in last if k != "setup_s"} | {"value": value, "unit": UNIT},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


KIND_NAMES = {1: "block_schur chebyshev-jacobi d=16 (kind 1)", 2: "block_reg, diag(M) Woodbury (kind 2)",
              3: "block_schur amg v-cycle on S_D (kind 3)",
              4: "block_schur amg v-cycle in FP32, FGMRES (kind 4, mixed precision)",
              5: "block_reg with the M-aware velocity block: PCG on M + B^T (eps W)^-1 B (kind 5)"}

PAPER_CONTEXT = {
    "note": "the paper's own timings: another machine, another space and BCs (context only, not a target)",
    "hardware": "INDACO cluster, 2 x Xeon E5-2683 v4 2.1 GHz per node, PETSc + MUMPS/GAMG over MPI (PAPER.md P:993-996)",
    "table1_cube_k1_435201_dofs": {"procs": 1, "block_schur": {"it": 66, "T_sol_s": 50},
                                   "block_reg": {"it": 84, "T_sol_s": 53}, "mumps_T_sol_s": 823,
                                   "cite": "PAPER.md P:1009-1014"},
    "table1_cube_k1_435201_dofs_p32": {"procs": 32, "block_schur": {"T_sol_s": 9},
                                       "block_reg": {"it": 137, "T_sol_s": 26}, "mumps_T_sol_s": 47,
                                       "cite": "PAPER.md P:1018"},
    "table4_cube_k2_804385_dofs_p8": {"procs": 8, "block_schur": {"it": 69, "T_sol_s": 217},
                                      "block_reg": {"it": 188, "T_sol_s": 87}, "cite": "PAPER.md P:1217"}}


def run_steps(solve, nsteps):
    """`nsteps` GMRES iterations: solves from x0 = 0 chained until the Arnoldi steps add up
    (each solve is capped at the steps still missing).  Returns the reports."""
    reps = []
    left = nsteps
    while left > 0:
        r = solve(left)
        reps.append(r)
        done = r["iterations"]
        if done <= 0:
            raise RuntimeError(f"solve made no progress: {r}")
        left -= done
    return reps


def check_full(rep, rtol, what):
    """ADVICE (round 1): never report a solve that hit maxit or broke down."""
    if not (rep["status"] == 0 and rep["converged"] == 1 and rep["rel_residual_true"] <= rtol * 1.0001):
        raise RuntimeError(f"{what}: solve did not converge: {rep}")


def secondary_c3(pkg, torch, steps=3):
    """C3 (round-1 headline) timed as whole solves: kind 3 (FP64 V-cycle) and kind 4 (FP32)."""
    from vemgen.configs import CONFIGS
    cfg = CONFIGS["C3"]
    s = cfg.build()
    sv = pkg.VemMixed(s.M, s.B, eps=0.0, layout=s.layout, opts=pkg.default_options(restart=cfg.restart))
    rhs = torch.from_numpy(s.rhs).cuda()
    out = {"workload": f"C3: {cfg.describe}", "n_dofs": s.n}
    for kind in (3, 4, 30, 40):
        if kind >= 30:   # kinds 3 / 4 with the compressed (float32) Krylov basis, SURVEY.md §8(f) N4
            sv.set_options(basis_f32=1)
            kind_arg = kind // 10
            label = KIND_NAMES[kind_arg] + ", float32-compressed Krylov basis (opts.basis_f32)"
        else:
            kind_arg, label = kind, KIND_NAMES[kind]
        for _ in range(2):
            sv.solve(rhs, cfg.rtol, 20000, kind_arg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = []
        a.record()
        for _ in range(steps):
            reps.append(sv.solve(rhs, cfg.rtol, 20000, kind_arg).report)
        b.record()
        torch.cuda.synchronize()
        for r in reps:
            check_full(r, cfg.rtol, f"C3 kind {kind}")
        ms = a.elapsed_time(b) / steps
        out[f"kind{kind_arg}_basis_f32" if kind >= 30 else f"kind{kind}"] = {
                              "precond": label, "time_to_solution_ms": round(ms, 2),
                              "iterations": reps[-1]["iterations"], "solves_per_s": round(1e3 / ms, 3),
                              "gmres_it_per_s": round(reps[-1]["iterations"] / (ms / 1e3), 1),
                              "rel_residual_true": reps[-1]["rel_residual_true"]}
    sv.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    import paper_1901_02330_b200 as pkg
    from vemgen.configs import CONFIGS, eps_for

    rank, ws, local = dist_init(args)
    torch.cuda.set_device(local)
    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    s = cfg.build()
    t_asm = time.perf_counter() - t0
    kind = headline_kind(cfg, s, args)
    eps = eps_for(s)
    nested = kind in (2, 5)
    # timed region: CUDA graphs with the sampled timing mode: one kernel launch per graph
    # replay is bracketed by CUDA events inside the graph (kinds 1/3: the middle Chebyshev /
    # fine-level smoother step of every Arnoldi step; kinds 2/5: one fine-level S_eps pass of the
    # inner V-cycle per replay of the inner-PCG graph): the live roofline of the dominant kernel
    # without per-launch overhead.  --per-launch: every launch timed, no graphs.
    timing = 1 if args.per_launch else 2
    opts = pkg.default_options(restart=cfg.restart, use_graphs=0 if args.per_launch else 1, timing=timing,
                               reorth=args.reorth, l2_persist=args.l2_persist)
    t0 = time.perf_counter()
    sv = pkg.VemMixed(s.M, s.B, eps=eps, layout=s.layout, opts=opts)
    t_up = time.perf_counter() - t0
    info = sv.info()
    rhs_dev = torch.from_numpy(s.rhs).cuda()
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def dev_solve(maxit):
        return sv.solve(rhs_dev, cfg.rtol, maxit, kind).report

    run_steps(dev_solve, max(args.warmup, 0))
    sv.kernel_stats(reset=True)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        reports = run_steps(dev_solve, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stats = sv.kernel_stats(reset=True)
    its = sum(r["iterations"] for r in reports)
    assert its == args.steps, (its, args.steps)
    # max over ranks of the time, sum of the work (every rank runs its own replica)
    ms, its_all = reduce_over_ranks(ms, its, device="cuda")
    value = its_all / (ms / 1e3)

    # end to end: host rhs (pinned) -> device -> solve -> u, p back to host, through the C ABI,
    # the same K steps; every solve call copies rhs in and u, p out
    rhs_pin = torch.from_numpy(s.rhs).pin_memory()
    u_pin = torch.empty(s.layout.n_u, dtype=torch.float64).pin_memory()
    p_pin = torch.empty(s.layout.n_p, dtype=torch.float64).pin_memory()
    sv.set_options(timing=0, use_graphs=1)

    def host_solve(maxit):
        return sv.solve_host(rhs_pin.numpy(), cfg.rtol, maxit, kind, u_pin.numpy(), p_pin.numpy()).report

    run_steps(host_solve, min(args.warmup, 2))
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e2e_reps = run_steps(host_solve, args.steps)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_ms, e2e_its = reduce_over_ranks(1e3 * e2e_s, sum(r["iterations"] for r in e2e_reps), device="cuda")
    e2e_calls = len(e2e_reps)

    # time to solution: ONE complete solve to rtol (the metric's first half); also the source
    # of the K / inner step counts per outer iteration that the oracle extrapolation uses
    sv.set_options(timing=0, use_graphs=1)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    full = sv.solve(rhs_dev, cfg.rtol, 20000, kind)
    f1.record(stream)
    torch.cuda.synchronize()
    check_full(full.report, cfg.rtol, f"{cfg.name} kind {kind}")
    fr = full.report
    tts_ms = f0.elapsed_time(f1)
    u, p = full.u.cpu().numpy(), full.p.cpu().numpy()
    conservation = float(np.abs(s.B @ u - s.f).max() / np.abs(s.f).max())
    counts = None
    if kind == 5 and fr["iterations"] > 1:
        real = fr["iterations"] - 1   # the first Krylov vector has no velocity part: no K solve
        counts = {"outer": fr["iterations"], "k_steps": fr["k_iterations"], "inner_steps": fr["inner_iterations"],
                  "k_per_outer": round(fr["k_iterations"] / real, 2),
                  "inner_per_k": round(fr["inner_iterations"] / max(fr["k_iterations"] + real, 1), 2)}
        if rank == 0:
            try:
                pth = os.path.join(ROOT, "profiles", "nested_counts.json")
                allc = json.load(open(pth)) if os.path.exists(pth) else {}
                allc[cfg.name] = counts
                json.dump(allc, open(pth, "w"), indent=1)
            except OSError:
                pass

    # kernel breakdown: a bounded run with every launch timed (after the timed region)
    sv.set_options(timing=1, use_graphs=0)
    nb_steps = min(args.steps, 4) if nested else 20000
    sv.kernel_stats(reset=True)
    rb = sv.solve(rhs_dev, cfg.rtol, nb_steps, kind)
    breakdown = sv.kernel_stats(reset=True)
    launches_per_it = sum(v["launches"] for v in breakdown.values()) / max(rb.report["iterations"], 1)

    hbm, peak_kind = peaks()
    per = {k: v for k, v in breakdown.items() if v["launches"]}
    tot_ms = max(sum(x["ms"] for x in per.values()), 1e-9)
    dom = max(per, key=lambda k: per[k]["ms"]) if per else None
    if kind == 5 and "mg_fine" in per:
        dom = "mg_fine"
    live = {k: v for k, v in stats.items() if v["launches"]}
    roof = None
    if dom:
        if dom in live:
            d = live[dom]
            src = "sampled CUDA events inside the timed region (graph event-record nodes around one launch per replay)"
        else:
            d = per[dom]
            src = "per-launch CUDA events, bounded breakdown run after the timed region"
        ach = d["bytes"] / (d["ms"] / 1e3) / 1e9
        agg = per[dom]
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "frac_of_nominal_8TBps": round(ach / 8000.0, 4),
                "traffic": ncu_traffic(dom), "peak_source": peak_kind,
                "bytes_per_launch": d["bytes"] / d["launches"], "avg_launch_us": 1e3 * d["ms"] / d["launches"],
                "launches_timed": d["launches"], "source": src,
                # the same class over every launch of the breakdown run, and its share of that run
                "class_aggregate": {"achieved": round(agg["bytes"] / (agg["ms"] / 1e3) / 1e9, 1),
                                    "frac": round(agg["bytes"] / (agg["ms"] / 1e3) / 1e9 / hbm, 4),
                                    "launches": agg["launches"], "share_of_run": round(agg["ms"] / tot_ms, 4),
                                    "source": "per-launch CUDA events, breakdown run"}}
    kern = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1),
                "frac_of_peak": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6 / hbm, 4),
                "share": round(v["ms"] / tot_ms, 4)}
            for k, v in per.items() if v["ms"] / tot_ms >= 1e-3}   # (gated no-op launches of a bounded run)

    secondary = None
    if rank == 0 and ws == 1 and not args.no_variant and cfg.name == "C5":
        sv.close()
        sv = None
        secondary = secondary_c3(pkg, torch)

    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "time_to_solution_ms": round(tts_ms, 2), "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded vemgen assembly, no dataset)",
            "config": {"workload": f"{cfg.name}: {cfg.describe}", "n_dofs": s.n, "n_u": s.layout.n_u,
                       "n_p": s.layout.n_p, "nnz_A": info["nnz_A"], "nnz_S": info["nnz_S"],
                       "precond": KIND_NAMES.get(kind, kind),
                       "step": "one GMRES iteration (preconditioner apply + saddle SpMV + batched CGS); the timed "
                               "region chains solves from x0 = 0, each capped at the steps still missing",
                       "solve_calls_in_timed_region": len(reports),
                       "inner_amg_levels": sv.inner_amg_levels() if (sv and nested) else None,
                       "restart": cfg.restart, "rtol": cfg.rtol,
                       "l2_window_MB": round(info["l2_window_bytes"] / 1e6, 1),
                       "orthogonalisation": {1: "CGS2", 0: "CGS1"}.get(args.reorth, "auto: CGS1 (GMRES) / CGS2 (FGMRES)"),
                       "setup_ms": fr["setup_ms"], "assembly_s": round(t_asm, 2),
                       "upload_wall_s": round(t_up, 2), "parallelism": f"replicas x{ws}",
                       "l2": "inputs larger than L2 (A %.0f MB, S_D %.0f MB, Krylov basis %.0f MB)" % (
                           12 * info["nnz_A"] / 1e6, 12 * info["nnz_S"] / 1e6,
                           8 * s.n * (cfg.restart + 1) * (2 if nested else 1) / 1e6),
                       "timing": ("CUDA graphs (GMRES cycles / inner-PCG chunks); sampled events" if not args.per_launch
                                  else "per-launch CUDA events, no graphs"),
                       "kernels_source": f"per-launch CUDA events over a bounded run ({rb.report['iterations']} "
                                         "GMRES iterations) after the timed region"},
            "full_solve": {"time_to_solution_ms": round(tts_ms, 2), "iterations": fr["iterations"],
                           "k_iterations": fr["k_iterations"], "inner_iterations": fr["inner_iterations"],
                           "restarts": fr["restarts"], "converged": fr["converged"],
                           "rel_residual_true": fr["rel_residual_true"], "conservation_rel": conservation,
                           "solves_per_s": round(1e3 / tts_ms, 5),
                           "gmres_it_per_s": round(fr["iterations"] / (tts_ms / 1e3), 4), "nested_counts": counts},
            "roofline": roof, "kernels": kern,
            "gpu_launches": int(round(launches_per_it * args.steps)),
            "secondary": secondary, "paper_context": PAPER_CONTEXT,
            "e2e": {"value": round(e2e_its / (e2e_ms / 1e3), 4), "unit": UNIT,
                    "ms_per_step": round(e2e_ms / args.steps, 3),
                    "h2d_bytes_per_step": 8 * s.n * e2e_calls / args.steps,
                    "d2h_bytes_per_step": 8 * s.n * e2e_calls / args.steps,
                    "solve_calls": e2e_calls,
                    "path": "vem_mixed_solve_host (pinned host rhs -> device, solve, u and p -> host; every call)"},
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(s, cfg, kind, eps, args.cpu_sample_its)
        line["cpu_baseline"].pop("setup_s", None)
    if sv:
        sv.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
