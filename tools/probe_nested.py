"""Bounded nested-solve probe (kinds 2 and 5): a few outer FGMRES steps of a config on
cuda:0, first untimed-per-launch (graphs on: wall time per outer step and the K / inner
step counts), then with every launch timed (per-class achieved bandwidth).
usage: probe_nested.py C5 5 2 [opt=value ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

name, kind, maxit = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
extra = {}
for a in sys.argv[4:]:
    k, v = a.split("=")
    extra[k] = float(v) if ("." in v or "e" in v) else int(v)
cfg = CONFIGS[name]
t0 = time.time()
s = cfg.build()
print(json.dumps({"assembly_s": round(time.time() - t0, 1), "n": s.n}), flush=True)
sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout, opts=pkg.default_options(restart=cfg.restart, **extra))
print(json.dumps({"info": sv.info(), "inner_levels": sv.inner_amg_levels()}), flush=True)
rhs = torch.from_numpy(s.rhs).cuda()
for timing in (0, 1):
    sv.set_options(timing=timing)
    sv.kernel_stats(reset=True)
    t0 = time.time()
    r = sv.solve(rhs, cfg.rtol, maxit, kind)
    wall = time.time() - t0
    rep = {k: r.report[k] for k in ("status_name", "iterations", "k_iterations", "inner_iterations",
                                    "rel_residual_true", "rel_residual_est", "solve_ms")}
    out = {"timing": timing, "wall_s": round(wall, 2), **rep}
    if timing:
        cl = {}
        for k, d in sv.kernel_stats(reset=True).items():
            if d["launches"]:
                cl[k] = {"launches": d["launches"], "ms": round(d["ms"], 1), "avg_us": round(1e3 * d["ms"] / d["launches"], 1),
                         "GBps": round(d["bytes"] / max(d["ms"], 1e-9) / 1e6, 1)}
        out["classes"] = cl
    print(json.dumps(out), flush=True)
sv.close()
