"""Parity at a config's stated size, run once and kept under profiles/ (too slow for the test
suite): the oracle's own full solve on the host cores against the GPU solve of the same system:
iterations, inner steps, ||.||_inf relative differences of u and p, true residual, conservation.
usage: full_parity.py C2:1 C2:2 C4:2 ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from oracle import solver as O  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

built = {}
for spec in sys.argv[1:]:
    name, kind = spec.split(":")
    kind = int(kind)
    cfg = CONFIGS[name]
    if name not in built:
        built.clear()
        built[name] = cfg.build()
    s = built[name]
    eps = eps_for(s)
    nb = s.layout.n_p_dof
    sv = pkg.VemMixed(s.M, s.B, eps=eps, layout=s.layout, opts=pkg.default_options(restart=cfg.restart))
    g = sv.solve(torch.from_numpy(s.rhs).cuda(), cfg.rtol, 20000, kind)
    u, p = g.u.cpu().numpy(), g.p.cpu().numpy()
    sv.close()
    t0 = time.time()
    ref = O.solve(s.M, s.B, s.rhs, kind, cfg.rtol, cfg.restart, eps=eps, block=nb)
    t_or = time.time() - t0
    nu = s.layout.n_u
    rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())  # noqa: E731
    x = np.concatenate([u, p])
    print(json.dumps({"config": name, "precond": kind, "n": s.n,
                      "gpu_iterations": g.report["iterations"], "oracle_iterations": ref.iterations,
                      "gpu_inner": g.report["inner_iterations"], "oracle_inner": int(ref.inner_iterations),
                      "rel_inf_u": rel(u, ref.x[:nu]), "rel_inf_p": rel(p, ref.x[nu:]),
                      "gpu_true_residual": float(np.linalg.norm(s.rhs - O.spmv_saddle(s.M, s.B, x)) / np.linalg.norm(s.rhs)),
                      "conservation_rel": float(np.abs(s.B @ u - s.f).max() / np.abs(s.f).max()),
                      "gpu_solve_ms": round(g.report["solve_ms"], 1), "oracle_solve_s": round(t_or, 1),
                      "oracle_converged": bool(ref.converged)}), flush=True)
