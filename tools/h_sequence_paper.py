"""E3 of the paper on its own space (Table 4: Cube meshes, k = 2, N_P = 512,
4096, 8000, 13824, 21952): paper-mode assembly (BDM-type space, pressure P_{k-1}; Dirichlet pressure
data instead of the paper's Neumann data + multiplier), both preconditioners with this build's
stand-ins for the MUMPS / GAMG inner solves, FGMRES/GMRES(50), rtol 1e-10.  One JSON line per (n, kind),
with the paper's own iteration count beside it.
Usage: python tools/h_sequence_paper.py [k] [n1,n2,...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import eps_for, paper_cube  # noqa: E402

PAPER_IT = {(2, 8): (113, 86), (2, 16): (78, 123), (2, 20): (76, 145), (2, 24): (72, 168), (2, 28): (69, 188),
            (1, 32): (66, 84)}   # (Block-Schur, Block-Reg) GMRES iterations, Tables 4 and 1
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ns = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "8,16,20,24,28").split(",")]
for n in ns:
    cfg = paper_cube(n, k)
    t0 = time.time()
    s = cfg.build()
    sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout, opts=pkg.default_options(restart=50))
    rhs = torch.from_numpy(s.rhs).cuda()
    kinds = [1, 2] + ([3] if s.layout.n_p_dof == 1 else [])
    for kind in kinds:
        r = sv.solve(rhs, 1e-10, 20000, kind).report
        paper = PAPER_IT.get((k, n))
        print(json.dumps({"k": k, "n": n, "N_P": n ** 3, "dofs": s.n, "paper_dofs": s.n + 1, "kind": kind,
                          "iterations": r["iterations"], "inner": r["inner_iterations"], "converged": r["converged"],
                          "solve_ms": round(r["solve_ms"], 1),
                          "paper_iterations": None if (paper is None or kind == 3) else paper[0 if kind == 1 else 1],
                          "assembly_s": round(time.time() - t0, 1)}), flush=True)
    sv.close()
