"""Small driver for compute-sanitizer: every entry point and preconditioner on
C1, C3s, C2s (k=1) and C4s (k=2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

for name in ("C1", "C3s", "C2s", "C4s"):
    cfg = CONFIGS[name]
    s = cfg.build()
    sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout, opts=pkg.default_options(restart=cfg.restart))
    x = torch.from_numpy(np.random.default_rng(0).normal(size=s.n)).cuda()
    sv.spmv(x)
    sv.schur_spmv(x[s.layout.n_u:].contiguous())
    kinds = (1, 2, 3) if s.layout.n_p_dof == 1 else (1, 2)
    for kind in kinds:
        sv.precond_apply(kind, x)
        r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 2000, kind)
        print(name, kind, r.report["status_name"], r.report["iterations"], flush=True)
    sv.solve_host(s.rhs, 1e-10, 2000, 1)
    sv.close()
print("sanitize_smoke done")
