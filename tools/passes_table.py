"""Print tools/gpu_passes.sh output: python tools/passes_table.py gpurun_out/c3_passes.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [n for n, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]
d = collections.OrderedDict()
for r in rows[i + 1:]:
    x = dict(zip(hdr, r))
    d.setdefault(x["ID"], {"kernel": x["Kernel Name"][:28]})[x["Metric Name"]] = x["Metric Value"]
for k, v in d.items():
    us = float(v["gpu__time_duration.sum"]) / 1e3
    gb = (float(v["dram__bytes_read.sum"]) + float(v["dram__bytes_write.sum"])) / 1e9
    print("%s %-28s %8.1f us  %6.3f GB  %6.0f GB/s  fmaH %5s%%  alu %5s%%  issue %5s%%" % (
        k, v["kernel"], us, gb, gb / us * 1e6,
        v.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "-"),
        v.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "-"),
        v.get("smsp__issue_active.avg.pct_of_peak_sustained_active", "-")))
