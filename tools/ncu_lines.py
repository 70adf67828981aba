"""Summarise an ncu report for one kernel: opcode mix and per-source-line instruction/stall shares.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top_n]
"""
import csv
import io
import os
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre,
                      "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
hdr = None
per_line, stall, per_op = Counter(), Counter(), Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ii:
        continue
    try:
        n = int(r[ii] or 0)
        smp = int(r[isamp] or 0)
    except ValueError:
        continue
    if r[0]:
        key = (f"{fname}:{r[0]}", r[1].strip()[:80])
        per_line[key] += n
        stall[key] += smp
    else:
        op = r[3].split()
        if op and op[0].startswith("@"):
            op = op[1:]
        if op:
            per_op[op[0].split(".")[0]] += n
tot = sum(per_op.values()) or 1
print("total warp instructions %.3e" % tot)
print("opcodes:", ", ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in per_op.most_common(16)))
tl = sum(per_line.values()) or 1
ts = sum(stall.values()) or 1
for (ln, src), v in per_line.most_common(top):
    print("%-22s %5.1f%% inst %5.1f%% stall  %s" % (ln, 100 * v / tl, 100 * stall[(ln, src)] / ts, src))
