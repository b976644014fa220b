"""Per-source-line executed instructions and stall samples from an ncu
source-page CSV (cuda,sass), aggregated over all listed launches.

    python tools/ncu_src_lines.py src.csv [min_pct] [n_elements]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
nel = float(sys.argv[3]) if len(sys.argv) > 3 else 0
cur = hdr = None
agg = collections.Counter()
samp = collections.Counter()
text = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r and hdr and r[0].isdigit():
        if len(r) > len(hdr):  # unescaped quotes in the source text split it
            extra = len(r) - len(hdr)
            r = [r[0], ",".join(r[1:2 + extra])] + r[2 + extra:]
        try:
            n, s = int(r[ii]), int(r[isamp])
        except ValueError:
            continue
        key = (cur, int(r[0]))
        agg[key] += n
        samp[key] += s
        text[key] = r[1][:80]
tot = sum(agg.values()) or 1
ts = sum(samp.values()) or 1
print("warp instructions %d%s" % (tot, ("  = %.0f thread-inst/element" % (tot * 32 / nel)) if nel else ""))
for key in sorted(agg):
    if 100 * agg[key] / tot >= minp or 100 * samp[key] / ts >= minp:
        extra = (" %6.1f/el" % (agg[key] * 32 / nel)) if nel else ""
        print("%-16s:%4d %5.1f%% inst %5.1f%% samp%s  %s" % (key[0], key[1], 100 * agg[key] / tot,
                                                      100 * samp[key] / ts, extra, text[key]))
