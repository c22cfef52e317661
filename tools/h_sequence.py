"""E3-style optimality check (Tables 4-6: iteration counts under
h-refinement) with this build's stand-ins: unit-cube grids, K = I, the sin source,
rtol 1e-10, GMRES(50), every preconditioner kind that applies.  One JSON line per
(k, n, kind): GMRES iterations, inner PCG steps, time to solution.
Usage: python tools/h_sequence.py [k:n1,n2,...] ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen import mesh as _mesh  # noqa: E402
from vemgen.assemble import build_system  # noqa: E402

specs = sys.argv[1:] or ["0:16,32,64,128", "1:8,16,32", "2:8,16,24,32"]
for spec in specs:
    k, ns = spec.split(":")
    k = int(k)
    for n in (int(v) for v in ns.split(",")):
        t0 = time.time()
        s = build_system(_mesh.cube_mesh(n), k)
        eps = 1e-6 * float(s.M.diagonal().mean())
        sv = pkg.VemMixed(s.M, s.B, eps=eps, layout=s.layout, opts=pkg.default_options(restart=50))
        rhs = torch.from_numpy(s.rhs).cuda()
        kinds = [1, 2] + ([3, 4] if k == 0 else [])
        for kind in kinds:
            r = sv.solve(rhs, 1e-10, 20000, kind).report
            print(json.dumps({"k": k, "n": n, "h": 1.0 / n, "dofs": s.n, "kind": kind, "iterations": r["iterations"],
                              "inner": r["inner_iterations"], "converged": r["converged"],
                              "solve_ms": round(r["solve_ms"], 2), "assembly_s": round(time.time() - t0, 1)}),
                  flush=True)
        sv.close()
