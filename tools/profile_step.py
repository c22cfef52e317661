"""Short driver for ncu: upload a config and run one bounded solve (maxit
Arnoldi steps) through the C ABI.  Used only for profiling captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 60
kind = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = CONFIGS[name]
kind = kind or cfg.precs[0]
s = cfg.build()
sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout,
                  opts=pkg.default_options(restart=cfg.restart, use_graphs=0))
r = sv.solve(torch.from_numpy(s.rhs).cuda(), cfg.rtol, maxit, kind)
torch.cuda.synchronize()
print("profile_step", name, r.report["iterations"], r.report["status_name"], sv.info())
