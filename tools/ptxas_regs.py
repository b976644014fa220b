"""Registers / spills / smem per kernel from nvcc -Xptxas -v logs (csrc/*.ptxas.log).

    python tools/ptxas_regs.py [pattern]
"""
import glob
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
for log in sorted(glob.glob("paper_1811_01490_b200/csrc/*.ptxas.log")):
    cur = None
    spill = ""
    for line in open(log):
        m = re.search(r"Compiling entry function '(\w+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = "spill %s/%s" % m.groups()
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            sm = re.search(r"(\d+) bytes smem", line)
            name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
            if pat in name:
                print("%4s regs  %6s smem  %-16s %s" % (m.group(1), sm.group(1) if sm else "0",
                                                       spill, name))
            cur = None
