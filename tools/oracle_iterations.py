"""Full-length oracle solves (CPU, oracle/ only) of the bench workloads: writes
profiles/oracle_iterations.json = {config: {precond kind: GMRES iterations to
rtol}}.  bench.py scales the oracle's bounded-sample iteration rate to solves/s
with these counts (the oracle's own, never the GPU's).
Usage: python tools/oracle_iterations.py C3:3 [C1:1 ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import solver as O  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "oracle_iterations.json")
table = json.load(open(OUT)) if os.path.exists(OUT) else {}
for spec in sys.argv[1:]:
    name, kind = spec.split(":")
    cfg = CONFIGS[name]
    s = cfg.build()
    t0 = time.perf_counter()
    r = O.solve(s.M, s.B, s.rhs, int(kind), cfg.rtol, cfg.restart, maxit=20000, eps=eps_for(s),
                block=s.layout.n_p_dof)
    dt = time.perf_counter() - t0
    table.setdefault(name, {})[kind] = {"iterations": r.iterations, "converged": bool(r.converged),
                                        "rel_residual_true": r.rel_residual_true, "wall_s": round(dt, 1)}
    print(name, kind, table[name][kind], flush=True)
    json.dump(table, open(OUT, "w"), indent=1, sort_keys=True)
