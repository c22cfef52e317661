"""Solve every BASELINE config (both preconditioners where the config names
them) on cuda:0 through the C ABI and print one JSON line per solve.
usage: run_configs.py C1,C2,C5:5,C4:1+2,C4:2:inner_precond=0 [maxit]
       (name[:kind+kind...[:option=value+option=value]]; C5 defaults to kind 5)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4", "C5"]
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
for spec in names:
    name, _, rest = spec.partition(":")
    ks, _, os_ = rest.partition(":")
    extra = {}
    for kv in (os_.split("+") if os_ else []):
        k_, v_ = kv.split("=")
        extra[k_] = float(v_) if ("." in v_ or "e" in v_) else int(v_)
    cfg = CONFIGS[name]
    t0 = time.time()
    s = cfg.build()
    t_asm = time.time() - t0
    sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout, opts=pkg.default_options(restart=cfg.restart, **extra))
    rhs = torch.from_numpy(s.rhs).cuda()
    kinds = list(cfg.precs) + ([3] if s.layout.n_p_dof == 1 and 1 in cfg.precs else [])
    if name.startswith("C5"):
        kinds = [5]   # the M-aware Block-Reg (R24); kind 2 stagnates on C5
    if ks:
        kinds = [int(k) for k in ks.split("+")]
    for kind in kinds:
        r = sv.solve(rhs, cfg.rtol, maxit, kind)
        u, p = r.u.cpu().numpy(), r.p.cpu().numpy()
        cons = float(np.abs(s.B @ u - s.f).max() / np.abs(s.f).max())
        rep = {k: r.report[k] for k in ("status_name", "iterations", "restarts", "inner_iterations",
                                        "k_iterations", "rel_residual_true", "setup_ms", "solve_ms")}
        print(json.dumps({"config": name, "precond": kind, "options": extra, "n": s.n, "assembly_s": round(t_asm, 1),
                          "conservation_rel": cons, **rep, "info": sv.info()}), flush=True)
    sv.close()
