"""Per-kernel-class achieved bandwidth of a bounded solve (every launch timed
with CUDA events, algorithmic bytes as the library counts them), for the
configs bench.py does not time (C2, C4, C5).  One JSON line per (config, kind).
Usage: python tools/kernel_roofline.py C5:2:40 C4:1:60 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_02330_b200 as pkg  # noqa: E402
from vemgen.configs import CONFIGS, eps_for  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
            os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6554.6


built = {}
for spec in sys.argv[1:]:
    name, kind, maxit = spec.split(":")
    kind, maxit = int(kind), int(maxit)
    cfg = CONFIGS[name]
    if name not in built:
        for v in built.values():
            v[1].close()
        built.clear()
        s = cfg.build()
        sv = pkg.VemMixed(s.M, s.B, eps=eps_for(s), layout=s.layout,
                          opts=pkg.default_options(restart=cfg.restart, use_graphs=0, timing=1))
        built[name] = (s, sv)
    s, sv = built[name]
    rhs = torch.from_numpy(s.rhs).cuda()
    sv.solve(rhs, cfg.rtol, min(maxit, 5), kind)          # warm-up
    sv.kernel_stats(reset=True)
    r = sv.solve(rhs, cfg.rtol, maxit, kind)
    st = sv.kernel_stats(reset=True)
    P = peak()
    out = {}
    for k, d in st.items():
        if d["launches"] == 0 or d["ms"] <= 0:
            continue
        gbs = d["bytes"] / (d["ms"] * 1e-3) / 1e9
        out[k] = {"launches": d["launches"], "avg_us": round(1e3 * d["ms"] / d["launches"], 2),
                  "MB_per_launch": round(d["bytes"] / d["launches"] / 1e6, 2),
                  "GBps": round(gbs, 1), "frac_measured_peak": round(gbs / P, 3)}
    print(json.dumps({"config": name, "kind": kind, "n": s.n, "iterations": r.report["iterations"],
                      "inner_iterations": r.report["inner_iterations"], "status": r.report["status_name"],
                      "peak_GBps": P, "classes": out, "info": sv.info()}), flush=True)
