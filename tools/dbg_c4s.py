import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_1901_02330_b200 as pkg
from vemgen import configs
s = configs.CONFIGS["C4s"].build()
sv = pkg.VemMixed(s.M, s.B, eps=configs.eps_for(s), layout=s.layout, opts=pkg.default_options(restart=50))
r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 2)
print(os.environ.get("VEM_PCG_SPLIT"), r.report["iterations"], r.report["inner_iterations"], sv.info()["reordered"])
sv = pkg.VemMixed(s.M, s.B, eps=configs.eps_for(s), layout=s.layout, opts=pkg.default_options(restart=50, reorder=0))
r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 10000, 2)
print("noreorder", r.report["iterations"], r.report["inner_iterations"])
