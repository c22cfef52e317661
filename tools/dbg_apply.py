import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1901_02330_b200 as pkg
from vemgen import configs
s = configs.CONFIGS[sys.argv[1]].build()
sv = pkg.VemMixed(s.M, s.B, eps=configs.eps_for(s), layout=s.layout)
v = np.random.default_rng(0).normal(size=s.n)
for kind in (1, 2):
    z, its = sv.precond_apply(kind, torch.from_numpy(v).cuda())
    torch.cuda.synchronize()
    print("kind", kind, "ok", float(z.abs().max()), its, flush=True)
