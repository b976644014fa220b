"""Pipe utilisation metrics (sm__pipe_*, sm__inst_executed_pipe_*) of the first
launch in an ncu raw-page CSV: python tools/ncu_pipes.py raw.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, r = rows[0], rows[1], rows[2]
for i, h in enumerate(hdr):
    if ("pipe" in h and ("pct" in h or "active" in h)) and r[i] not in ("", "n/a"):
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        if v > 0.5:
            print("%-90s %10.2f %s" % (h, v, units[i]))
