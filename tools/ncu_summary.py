"""Summaries of ncu artefacts (run here, on the CPU box).
  python tools/ncu_summary.py launches <csv>      per-kernel share of a launch list
  python tools/ncu_summary.py report <ncu-rep>    key metrics of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if not (name.startswith("gcol::") or "::k_" in name or name.startswith("k_")):
            continue  # not ours (e.g. torch kernels of the graph generator)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(t for _, t in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:70]:70s} n={c:4d} total={t / 1e3:10.1f}us avg={t / c / 1e3:9.2f}us "
                   f"share={100 * t / tot:5.1f}%")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_op_read.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_no_instructions",
        "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_sample_count"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    lines = []
    for r in rows[2:]:
        lines.append(f"kernel: {r[h.index('Kernel Name')][:100]}")
        for k in KEYS:
            if k in h:
                lines.append(f"  {k} = {r[h.index(k)]} {rows[1][h.index(k)]}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(launches(sys.argv[2]) if sys.argv[1] == "launches" else report(sys.argv[2]))
