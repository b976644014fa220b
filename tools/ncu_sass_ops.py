"""Executed-instruction histogram per SASS opcode (and stall samples) from an
ncu source page exported with --print-source sass.

    python tools/ncu_sass_ops.py sass.csv [n_elements]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nel = float(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr = None
ops = collections.Counter()
samp = collections.Counter()
stall_cols = {}
stalls = collections.Counter()
for r in rows:
    if r and "Source" in r and "Instructions Executed" in r:
        hdr = r
        isrc = hdr.index("Source")
        iinst = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
        stall_cols = {i: h for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h}
        continue
    if not hdr or len(r) < len(hdr):
        continue
    try:
        n = int(r[iinst] or 0)
    except ValueError:
        continue
    txt = r[isrc].strip()
    toks = txt.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    ops[op] += n
    if isamp is not None:
        try:
            samp[op] += int(r[isamp] or 0)
        except ValueError:
            pass
tot = sum(ops.values()) or 1
ts = sum(samp.values()) or 1
print("warp instructions %d%s" % (tot, ("  = %.0f thread-inst/element" % (tot * 32 / nel)) if nel else ""))
fam = collections.Counter()
for op, n in ops.items():
    fam[op.split(".")[0]] += n
print("-- by family")
for op, n in fam.most_common(20):
    print("%-10s %6.2f%%%s" % (op, 100 * n / tot, (" %7.1f/el" % (n * 32 / nel)) if nel else ""))
print("-- by opcode")
for op, n in ops.most_common(45):
    print("%-28s %6.2f%% inst %5.1f%% samp%s" % (op, 100 * n / tot, 100 * samp[op] / ts,
                                                 (" %7.1f/el" % (n * 32 / nel)) if nel else ""))
