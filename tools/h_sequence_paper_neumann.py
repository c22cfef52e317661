"""E3 of the paper on its own problem (Table 4: Cube meshes, k = 2, N_P = 512 ..
21952; Table 1: 32768 cubes at k = 1): BDM-type space, nu = 1, the polynomial solution of P:898-911,
Neumann data on the whole boundary and the mean-value multiplier (vemgen.configs.paper_neumann;
the multiplier in closed form, the consistent singular saddle system through the C ABI, the
pressure projected onto mean zero), both preconditioners, GMRES/FGMRES(50), rtol 1e-10.  One JSON
line per (n, kind) with the paper's own iteration count beside it and the errors e_u, e_p.
Usage: python tools/h_sequence_paper_neumann.py [k] [n1,n2,...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen import assemble  # noqa: E402
from vemgen.configs import paper_neumann  # noqa: E402

PAPER_IT = {(2, 8): (113, 86), (2, 16): (78, 123), (2, 20): (76, 145), (2, 24): (72, 168), (2, 28): (69, 188),
            (1, 32): (66, 84)}   # (Block-Schur, Block-Reg) GMRES iterations, Tables 4 and 1
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ns = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "8,16,20,24,28").split(",")]
for n in ns:
    t0 = time.time()
    s, N = paper_neumann(n, k)
    eps = 1e-6 * float(N.M.diagonal().mean())
    sv = pkg.VemMixed(N.M, N.B, eps=eps, layout=s.layout, opts=pkg.default_options(restart=50))
    rhs = torch.from_numpy(N.rhs).cuda()
    for kind in (1, 2):
        res = sv.solve(rhs, 1e-10, 20000, kind)
        r = res.report
        u, p = res.u.cpu().numpy(), N.project(res.p.cpu().numpy())
        old = assemble.exact_u, assemble.exact_p
        assemble.exact_u = lambda pts, K=None: assemble.paper_exact_u(pts)
        assemble.exact_p = lambda pts: assemble.paper_exact_p(pts) - assemble.PAPER_P_MEAN
        try:
            eu, ep = assemble.l2_errors(s, u, p)
        finally:
            assemble.exact_u, assemble.exact_p = old
        paper = PAPER_IT.get((k, n))
        print(json.dumps({"k": k, "n": n, "N_P": n ** 3, "dofs_with_multiplier": s.n + 1, "kind": kind,
                          "iterations": r["iterations"], "inner": r["inner_iterations"], "converged": r["converged"],
                          "solve_ms": round(r["solve_ms"], 1), "e_u": float(eu), "e_p": float(ep),
                          "multiplier": N.lam, "mean_p": float(N.c @ p),
                          "paper_iterations": None if paper is None else paper[0 if kind == 1 else 1],
                          "assembly_s": round(time.time() - t0, 1)}), flush=True)
    sv.close()
