"""Aggregate an ncu source-page CSV (--page source --csv --print-source cuda,sass)
per CUDA source line: stall samples and executed warp instructions.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur = None
out = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = r
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        iinst = hdr.index("Instructions Executed")
        continue
    if r and hdr and r[0].isdigit():
        try:
            s, n = int(r[isamp]), int(r[iinst])
        except (ValueError, IndexError):
            continue
        if s or n:
            out.append((s, n, cur, r[0], r[1][:90]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("total stall samples", ts, "warp instructions", ti)
for o in sorted(out, reverse=True)[:top]:
    print("%5.1f%% samples %5.1f%% inst  %s:%s  %s" % (100 * o[0] / ts, 100 * o[1] / ti, o[2], o[3], o[4]))
