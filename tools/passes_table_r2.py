"""Per-pass ncu table (time, DRAM bytes, instructions per element, pipe %,
occupancy, top stall) from tools/ncu_summary.py 'full' outputs.

    python tools/passes_table_r2.py <metrics.txt> <elements per launch> [label]
"""
import re
import sys


def parse(path):
    launches, cur = [], None
    for ln in open(path):
        if ln.startswith("launch"):
            cur = {"name": ln.split(" ", 2)[2].strip(), "stalls": {}}
            launches.append(cur)
            continue
        parts = ln.split()
        if not parts or cur is None:
            continue
        if parts[0] == "stall":
            m = re.search(r"stalled_(\w+?)_per_issue", parts[1])
            cur["stalls"][m.group(1)] = float(parts[2])
        else:
            try:
                cur[parts[0]] = float(parts[1])
            except (ValueError, IndexError):
                pass
    return launches


def main():
    path, nel = sys.argv[1], float(sys.argv[2])
    label = sys.argv[3] if len(sys.argv) > 3 else path
    print("# %s: ncu --set full --clock-control none, one launch per pass" % label)
    print("| pass | kernel | ms | DRAM GB (r+w) | DRAM TB/s | thread-inst/element | issue % | "
          "warps active % | ALU pipe % | FMA pipe % | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for i, L in enumerate(parse(path)):
        ms = L.get("gpu__time_duration.sum", 0) / (1e3 if L.get("gpu__time_duration.sum", 0) > 50 else 1)
        gb = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
        ipe = L.get("smsp__inst_executed.sum", 0) * 32 / nel
        top = sorted(((v, k) for k, v in L["stalls"].items() if k != "selected"), reverse=True)[:3]
        print("| %d | %s | %.4f | %.3f | %.2f | %.0f | %.1f | %.1f | %.1f | %.1f | %s |" % (
            i, L["name"], ms, gb, gb / ms if ms else 0, ipe,
            L.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
            L.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
            L.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 0),
            L.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 0),
            ", ".join("%s %.2f" % (k, v) for v, k in top)))


if __name__ == "__main__":
    main()
