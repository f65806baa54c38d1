"""Summarise ncu outputs for profiles/ (run here, on the CPU side, after a gpurun call).

    python tools/ncu_summary.py launches gpurun_out/launches_X.csv   # per-kernel share of a step
    python tools/ncu_summary.py full gpurun_out/prof_X.ncu-rep       # key metrics of a --set full capture
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
        name = name.split("(")[0].split("<")[0]
        try:
            v = float(r[mi].replace(",", ""))
        except ValueError:
            continue
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot/1e3:.1f} us total (ncu, serialised, cold)",
           f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'us/launch':>10s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:44s} {v[0]:8d} {v[1]/1e3:10.1f} {v[1]/1e3/v[0]:10.2f} {100*v[1]/tot:5.1f}%")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "launch__cluster_dim_x", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__inst_executed.sum"]


def full(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    h, units = rows[0], rows[1]
    out = [f"# {path}"]
    for row in rows[2:]:
        out.append(f"## {row[h.index('Kernel Name')][:120]}")
        for w in WANT:
            if w in h:
                out.append(f"  {w:62s} {row[h.index(w)]:>16s} {units[h.index(w)]}")
        if "dram__bytes_read.sum" in h:
            pass
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
