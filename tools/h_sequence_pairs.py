"""E3-style optimality check (Tables 4-6: Block-Reg iteration counts under
h-refinement) on the C5 family: n^3 cubes with ~50% seeded pairs, k = 1, K = diag(1,1,1e-2) x
checkerboard {1, 1e-3} on (n/8)^3-cube blocks (8 blocks per axis, as C5), precond kind 5,
FGMRES(50), rtol 1e-10.  One JSON line per n: outer iterations, K steps, inner steps, time.
Usage: python tools/h_sequence_pairs.py [n1,n2,...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import Config, eps_for  # noqa: E402

ns = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,16,24,32,48,64").split(",")]
for n in ns:
    cfg = Config(f"P{n}", "pairs", n, 1, (2,), 50, block=max(n // 8, 1), seed=5)
    t0 = time.time()
    s = cfg.build()
    sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout, opts=pkg.default_options(restart=50))
    r = sv.solve(torch.from_numpy(s.rhs).cuda(), 1e-10, 3000, pkg.PRECOND_BLOCK_REG_M).report
    print(json.dumps({"n": n, "h": 1.0 / n, "dofs": s.n, "kind": 5, "iterations": r["iterations"],
                      "k_iterations": r["k_iterations"], "inner": r["inner_iterations"], "converged": r["converged"],
                      "rel_residual_true": r["rel_residual_true"], "solve_ms": round(r["solve_ms"], 1),
                      "inner_levels": sv.inner_amg_levels(), "assembly_s": round(time.time() - t0, 1)}), flush=True)
    sv.close()
