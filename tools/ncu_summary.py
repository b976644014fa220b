"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches <launches.csv>     per-kernel launch totals
    python tools/ncu_summary.py full <prof.ncu-rep>          key --set full metrics per launch
"""
import collections
import csv
import io
import re
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread",
    "launch__block_size",
    "launch__grid_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_not_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_dispatch_stall_per_warp_active.pct",
    "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct",
    "smsp__warp_issue_stalled_drain_per_warp_active.pct",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [n for n, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    print("%6s %12s %6s  %s" % ("count", "total_us", "share", "kernel"))
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%6d %12.1f %5.1f%%  %s" % (a[0], a[1] / 1e3, 100 * a[1] / tot, k))


def full(path):
    if path.endswith(".csv"):  # a raw page already exported on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("launch %s %s" % (d.get("ID"), re.sub(r"\(.*", "", d.get("Kernel Name", ""))))
        for m in FULL_METRICS:
            if m in d:
                print("  %-60s %s" % (m, d[m]))
        # warp-state breakdown (stall reasons, cycles per issued instruction)
        st = []
        for m, v in d.items():
            if m.startswith("smsp__average_warp_latency_issue_stalled_") or (
                    m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio")):
                try:
                    st.append((float(v.replace(",", "")), m))
                except ValueError:
                    pass
        for v, m in sorted(st, reverse=True)[:12]:
            if v > 0.01:
                print("  stall %-70s %s" % (m, v))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
