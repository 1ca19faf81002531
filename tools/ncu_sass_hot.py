#!/usr/bin/env python
"""Dynamic SASS census from an ncu source page export (--page source --csv --print-source sass).

usage: python tools/ncu_sass_hot.py <source.csv> [warp_chunks]
Prints executed warp instructions by opcode (and per warp-chunk if the number of
32-row warp-chunks of the launch is given), plus the top stall-sampled lines.
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
chunks = float(sys.argv[2]) if len(sys.argv) > 2 else 0
ops, samp = Counter(), Counter()
tot = 0
lines = []
for r in rows[hdr_i + 1:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    n = int(r[ie])
    t = re.sub(r"^@!?U?P\w+\s+", "", r[src].strip())
    op = t.split()[0] if t else "?"
    ops[op] += n
    samp[op] += int(r[ss] or 0)
    tot += n
    lines.append((n, int(r[ss] or 0), r[0], r[src].strip()))
print("total warp instructions", tot, ("per warp-chunk %.1f" % (tot / chunks)) if chunks else "")
for op, n in ops.most_common(45):
    print(f"{n:10d} {n / chunks if chunks else 0:8.1f} {samp[op]:7d} {op}")
