#!/usr/bin/env python
"""Benchmark of the hot path: block-preconditioned GMRES on the mixed-VEM
saddle-point system (BASELINE.json metric: time-to-solution & GMRES iters/s at
1 B200; SpMV / preconditioner HBM GB/s vs peak).

One step = one vem_mixed_solve of the configured system from x0 = 0 to
rtol 1e-10 (upload and S_D build happen once, before timing: reported as
setup_ms).  value = solves / s over the K timed steps, all ranks (the inverse of
the time to solution, summed over replicas); the GMRES iteration rate is reported
beside it (gmres_it_per_s), as are the per-kernel HBM rates.

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
UNIT = "solves/s"
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
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
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


def cpu_baseline(system, cfg, kind, eps, its):
    """The oracle as it stands on a bounded sample: `its` GMRES iterations of the
    same system on the host cores."""
    import numpy as np
    from oracle import solver as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = 1
    t0 = time.perf_counter()
    P = O.Preconditioner(kind, system.M, system.B, eps=eps, block=system.layout.n_p_dof)
    t1 = time.perf_counter()
    res = O.gmres(lambda x: O.spmv_saddle(system.M, system.B, x), P.apply, system.rhs, 1e-10, cfg.restart, its,
                  P.flexible, 1 if P.flexible else 0)
    t2 = time.perf_counter()
    itps = res.iterations / (t2 - t1)
    full = oracle_iterations(cfg.name, kind)
    return {"value": (itps / full) if full else None, "unit": UNIT, "cores": int(cores), "kind": "oracle",
            "gmres_it_per_s": itps, "iterations_per_solve": full,
            "sample": f"{res.iterations} GMRES iterations of {cfg.name} (precond {kind}) from x0=0, "
                      f"{t2 - t1:.1f} s (+{t1 - t0:.1f} s preconditioner setup, untimed); solves/s = "
                      f"it/s / {full} (the oracle's own full-solve count, profiles/oracle_iterations.json)",
            "setup_s": t1 - t0}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (rank 0 only)."""
    rank, ws, _ = dist_init(args)
    if rank != 0:
        return
    from vemgen.configs import CONFIGS, eps_for
    cfg = CONFIGS[args.config]
    s = cfg.build()
    kind = headline_kind(cfg, s, args)   # the same preconditioner as our arm
    eps = eps_for(s)
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(s, cfg, kind, eps, 1)
    t0 = time.perf_counter()
    tot_its = 0
    last = None
    for _ in range(args.steps):
        last = cpu_baseline(s, cfg, kind, eps, args.cpu_sample_its)
        vals.append(last["value"])
        tot_its += args.cpu_sample_its
    dt = time.perf_counter() - t0
    value = sum(vals) / len(vals) if all(v is not None for v in vals) else None
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded vemgen assembly)",
            "config": {"workload": f"{cfg.name}: {cfg.describe}", "rtol": cfg.rtol, "restart": cfg.restart,
                       "precond": kind, "n_dofs": s.n},
            "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample", "gmres_it_per_s", "iterations_per_solve")}
            | {"value": value, "unit": UNIT},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    # the same system assembled on the device (N2: element-parallel, shape-cached classes);
    # the solve below uses the host system (the definition the oracle shares)
    dev_asm = None
    try:
        from vemgen.assemble import class_templates
        t0 = time.perf_counter()
        tm = class_templates(cfg.make_mesh(), cfg.k)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        a = pkg.Assembled(tm, s.layout.n_u, s.layout.n_p)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        dev_asm = {"shape_cache_s": round(t1 - t0, 3), "device_s": round(t3 - t2, 3),
                   "nnz_equal": a.nnz() == (s.M.nnz, s.B.nnz)}
        a.close()
    except ValueError:
        pass
    # timed region: CUDA graphs (one graph launch per GMRES cycle) with the
    # sampled timing mode: the middle Chebyshev step of every Arnoldi step is
    # bracketed by CUDA events inside the graph (live roofline of the dominant
    # kernel without per-launch overhead).  --per-launch: every launch timed.
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

    for _ in range(args.warmup):
        r = sv.solve(rhs_dev, cfg.rtol, 20000, kind)
    sv.kernel_stats(reset=True)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reports = []
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = sv.solve(rhs_dev, cfg.rtol, 20000, kind)
            reports.append(r.report)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stats = sv.kernel_stats(reset=True)
    its = sum(r["iterations"] for r in reports)
    # max over ranks of the time, sum of the work
    ms, its_all = reduce_over_ranks(ms, its, device="cuda")
    solves_all = float(args.steps * ws)   # every rank solves its own replica K times
    value = solves_all / (ms / 1e3)
    it_rate = its_all / (ms / 1e3)

    # kernel breakdown: one more solve with every launch timed (after the timed region)
    sv.set_options(timing=1, use_graphs=0)
    rb = sv.solve(rhs_dev, cfg.rtol, 20000, kind)
    breakdown = sv.kernel_stats(reset=True)
    launches_per_solve = int(sum(v["launches"] for v in breakdown.values()))

    # end to end: host rhs (pinned) -> device -> solve -> u, p back to host, through the C ABI
    rhs_pin = torch.from_numpy(s.rhs).pin_memory()
    u_pin = torch.empty(s.layout.n_u, dtype=torch.float64).pin_memory()
    p_pin = torch.empty(s.layout.n_p, dtype=torch.float64).pin_memory()
    sv.set_options(timing=0, use_graphs=1)
    sv.solve_host(rhs_pin.numpy(), cfg.rtol, 20000, kind, u_pin.numpy(), p_pin.numpy())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_its = 0
    for _ in range(args.steps):
        rh = sv.solve_host(rhs_pin.numpy(), cfg.rtol, 20000, kind, u_pin.numpy(), p_pin.numpy())
        e2e_its += rh.report["iterations"]
    e2e_s = time.perf_counter() - t0
    e2e_graph_its = e2e_its

    # variants of the same approximate-Schur preconditioner, timed the same way:
    # kind 1 (fixed-sweep Chebyshev-Jacobi on S_D) and kind 4 (the V-cycle in FP32 inside
    # FP64 FGMRES) beside the kind-3 headline
    names = {1: "block_schur chebyshev-jacobi d=16 (kind 1)", 3: "block_schur amg v-cycle (kind 3)",
             4: "block_schur amg v-cycle in FP32, FGMRES (kind 4, mixed precision)"}
    variants = []
    vkinds = {3: [pkg.PRECOND_BLOCK_SCHUR, pkg.PRECOND_BLOCK_SCHUR_AMG_F32],
              1: [pkg.PRECOND_BLOCK_SCHUR_AMG]}.get(kind, [])
    for vkind in (vkinds if info.get("amg_levels", 0) > 0 and not args.no_variant else []):
        sv.set_options(timing=0, use_graphs=1)
        sv.solve(rhs_dev, cfg.rtol, 20000, vkind)
        torch.cuda.synchronize()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        vrep = []
        v0.record(stream)
        for _ in range(args.steps):
            vrep.append(sv.solve(rhs_dev, cfg.rtol, 20000, vkind).report)
        v1.record(stream)
        torch.cuda.synchronize()
        vms = v0.elapsed_time(v1) / args.steps
        variants.append({"precond": names[vkind], "time_to_solution_ms": round(vms, 2),
                         "iterations_per_solve": [r["iterations"] for r in vrep],
                         "GMRES_it_per_s": round(sum(r["iterations"] for r in vrep) / (args.steps * vms / 1e3), 2),
                         "rel_residual_true": vrep[-1]["rel_residual_true"]})
    variant = variants or None

    # SURVEY.md §8(d) Q21 benchmark extra: the same matrices with a seeded N(0, 1) RHS (seed 7)
    random_rhs = None
    if not args.no_variant:
        from vemgen.configs import random_rhs as _rr
        rr_dev = torch.from_numpy(_rr(s.n)).cuda()
        sv.set_options(timing=0, use_graphs=1)
        sv.solve(rr_dev, cfg.rtol, 20000, kind)
        torch.cuda.synchronize()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qrep = []
        q0.record(stream)
        for _ in range(args.steps):
            qrep.append(sv.solve(rr_dev, cfg.rtol, 20000, kind).report)
        q1.record(stream)
        torch.cuda.synchronize()
        qms = q0.elapsed_time(q1) / args.steps
        random_rhs = {"rhs": "N(0,1), seed 7 (vemgen.configs.random_rhs)", "precond": kind,
                      "time_to_solution_ms": round(qms, 2),
                      "iterations_per_solve": [r["iterations"] for r in qrep],
                      "GMRES_it_per_s": round(sum(r["iterations"] for r in qrep) / (args.steps * qms / 1e3), 2),
                      "rel_residual_true": qrep[-1]["rel_residual_true"]}

    hbm, peak_kind = peaks()
    per = {k: v for k, v in breakdown.items() if v["launches"]}
    dom = max(per, key=lambda k: per[k]["ms"]) if per else None
    # the dominant kernel's live numbers come from the timed region when sampled
    live = {k: v for k, v in stats.items() if v["launches"]}
    if dom in live:
        per_dom = live[dom]
        dom_src = ("sampled CUDA events inside the timed region (" +
                   ("fine-level pre-smoothing step of the V-cycle" if kind == 3 else "middle Chebyshev step") +
                   " of every Arnoldi step)")
    else:
        per_dom = per.get(dom)
        dom_src = "per-launch CUDA events, breakdown solve after the timed region"
    roof = None
    if dom:
        d = per_dom
        ach = d["bytes"] / (d["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": ncu_traffic(dom), "peak_source": peak_kind,
                "bytes_per_launch": d["bytes"] / d["launches"], "avg_launch_us": 1e3 * d["ms"] / d["launches"],
                "launches_timed": d["launches"], "source": dom_src}
    kern = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1),
                "share": round(v["ms"] / max(sum(x["ms"] for x in per.values()), 1e-9), 4)}
            for k, v in per.items()}
    launches = launches_per_solve * args.steps
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "time_to_solution_ms": round(ms / args.steps, 2),
            "gmres_it_per_s": round(it_rate, 1), "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded vemgen assembly, no dataset)",
            "config": {"workload": f"{cfg.name}: {cfg.describe}", "n_dofs": s.n, "n_u": s.layout.n_u,
                       "n_p": s.layout.n_p, "nnz_A": info["nnz_A"], "nnz_S": info["nnz_S"],
                       "precond": {1: "block_schur chebyshev-jacobi d=16 (kind 1)", 2: "block_reg (kind 2)",
                                   3: "block_schur amg v-cycle on S_D (kind 3)"}.get(kind, kind),
                       "amg_levels": sv.amg_levels() if kind == 3 else None,
                       "restart": cfg.restart, "rtol": cfg.rtol,
                       "l2_window_MB": round(info["l2_window_bytes"] / 1e6, 1),
                       "orthogonalisation": {1: "CGS2", 0: "CGS1"}.get(args.reorth, "auto: CGS1 (GMRES) / CGS2 (FGMRES)"),
                       "iterations_per_solve": [r["iterations"] for r in reports],
                       "time_to_solution_ms": ms / args.steps,
                       "rel_residual_true": reports[-1]["rel_residual_true"],
                       "setup_ms": reports[-1]["setup_ms"], "assembly_s": round(t_asm, 2),
                       "device_assembly": dev_asm,
                       "upload_wall_s": round(t_up, 2), "parallelism": f"replicas x{ws}",
                       "l2": "inputs larger than L2 (A %.0f MB + Krylov basis %.0f MB)" % (
                           (12 * info["nnz_A"]) / 1e6, 8 * s.n * (cfg.restart + 1) / 1e6),
                       "timing": ("CUDA graphs, one graph per GMRES cycle; sampled events" if not args.per_launch
                                  else "per-launch CUDA events, no graphs"),
                       "kernels_source": "per-launch CUDA events over one extra solve after the timed region"},
            "roofline": roof, "kernels": kern, "gpu_launches": launches, "variant": variant,
            "random_rhs": random_rhs,
            "e2e": {"value": round(args.steps / e2e_s, 3), "unit": UNIT, "time_to_solution_ms": round(1e3 * e2e_s / args.steps, 2),
                    "gmres_it_per_s": round(e2e_graph_its / e2e_s, 1),
                    "h2d_bytes_per_step": 8 * s.n, "d2h_bytes_per_step": 8 * s.n,
                    "path": "vem_mixed_solve_host (pinned host rhs -> solve -> u, p to host), CUDA graphs"},
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(s, cfg, kind, eps, args.cpu_sample_its)
        line["cpu_baseline"].pop("setup_s", None)
    sv.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
