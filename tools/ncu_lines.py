"""Aggregate an ncu source-page CSV (--print-source cuda,sass) per CUDA line
for the first profiled kernel: stall samples and executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur = None
out = []
hdr = None
seen = set()
for r in rows:
    if r and r[0] == "File Path":
        if r[1] in seen:
            break
        seen.add(r[1])
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0] not in ("", "Function Name") and hdr:
        try:
            out.append((int(r[4]), int(r[7]), cur, r[0], r[1][:80]))
        except ValueError:
            pass
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("total stall samples", ts, "warp instructions", ti)
for o in sorted(out, reverse=True)[:top]:
    print("%5.1f%% samples %5.1f%% inst  %s:%s  %s" % (100 * o[0] / ts, 100 * o[1] / ti, o[2], o[3], o[4]))
