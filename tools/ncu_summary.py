"""Summarise ncu outputs into profiles/: launch list (csv) -> per-kernel table,
and a --set full report -> per-kernel key metrics.  Run here (no GPU needed)."""
import collections
import csv
import io
import subprocess
import sys


def launches(path, out, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in data:
        per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0, 0.0])
    for (_, k), m in per.items():
        name = k.split("(")[0].split("<")[0]
        t = m.get("gpu__time_duration.sum", 0)
        a = agg[name]
        a[0] += 1
        a[1] += t
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        if t > 5000:
            a[3] += 1
            a[2] += b
            a[4] += t
    tot = sum(a[1] for a in agg.values())
    lines = [f"# {title}", "# cold-cache serialised per-launch ncu times: compare SHARES with bench.py, not absolutes;",
             "# 'active' = launches > 5 us (gated launches after the step cap early-exit in ~2 us)",
             "kernel,launches,active_launches,total_us,share,avg_active_us,dram_MB_per_active_launch,active_dram_GBps"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        act = max(a[3], 1)
        lines.append(f"{k},{a[0]},{a[3]},{a[1] / 1e3:.1f},{a[1] / tot:.4f},{a[4] / act / 1e3:.1f},"
                     f"{a[2] / act / 1e6:.1f},{a[2] / max(a[4], 1):.0f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "launch__occupancy_limit_registers"]


def full(rep, out, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, data = rows[0], rows[1], rows[2:]
    lines = [f"# {title}", "kernel," + ",".join(f"{k} ({u[h.index(k)]})" for k in KEYS if k in h) + ",traffic_MB"]
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0]
        vals = [r[h.index(k)] for k in KEYS if k in h]
        tr = float(r[h.index("dram__bytes_read.sum")]) + float(r[h.index("dram__bytes_write.sum")])
        lines.append(name + "," + ",".join(vals) + f",{tr:.1f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    kind, src, out, title = sys.argv[1:5]
    (launches if kind == "launches" else full)(src, out, title)
