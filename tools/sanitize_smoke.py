"""Small driver for compute-sanitizer: every entry point and preconditioner on
C1, C3s, C2s (k=1), C4s (k=2) and the C5-type C5t (kind 5); both inner-PCG forms.
  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

for name in ("C1", "C3s", "C2s", "C4s", "C5t"):
    cfg = CONFIGS[name]
    s = cfg.build()
    sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout, opts=pkg.default_options(restart=cfg.restart))
    x = torch.from_numpy(np.random.default_rng(0).normal(size=s.n)).cuda()
    sv.spmv(x)
    sv.schur_spmv(x[s.layout.n_u:].contiguous())
    kinds = (1, 2, 3, 4, 5) if s.layout.n_p_dof == 1 else (1, 2, 5)
    for kind in kinds:
        sv.precond_apply(kind, x)
        # bounded where the default tolerances are not meant to converge (kind 2 on the C5 type;
        # kind 5 with k_inner_rtol = 1e-8 on the tets / k = 2 cubes, R24)
        cap = 40 if ((name == "C5t" and kind == 2) or (kind == 5 and name in ("C2s", "C4s"))) else 2000
        r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, cap, kind)
        print(name, kind, r.report["status_name"], r.report["iterations"], flush=True)
    sv.set_options(inner_precond=0)
    r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 40, 2)
    print(name, "2 (block-Jacobi inner PCG)", r.report["status_name"], r.report["iterations"], flush=True)
    sv.solve_host(s.rhs, 1e-10, 2000, 1)
    sv.close()
print("sanitize_smoke done")
