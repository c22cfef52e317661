"""A/B of the compressed (float32) Krylov basis on C3 (opts.basis_f32):
time to solution and iterations of kinds 3, 4 and 1 with the FP64 and the compressed basis."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["C3"]
s = cfg.build()
sv = pkg.VemMixed(s.M, s.B, eps=0.0, layout=s.layout, opts=pkg.default_options(restart=50))
rhs = torch.from_numpy(s.rhs).cuda()
for b32 in (0, 1, 0, 1):
    sv.set_options(basis_f32=b32)
    for kind in (3, 4, 1):
        sv.solve(rhs, 1e-10, 20000, kind)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            r = sv.solve(rhs, 1e-10, 20000, kind)
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"config": "C3", "basis_f32": b32, "kind": kind, "iterations": r.report["iterations"],
                          "time_to_solution_ms": round(a.elapsed_time(b) / 3, 2),
                          "rel_residual_true": r.report["rel_residual_true"]}), flush=True)
sv.close()
