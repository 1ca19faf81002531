#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples from an ncu report.

usage: python tools/ncu_lines.py <report.ncu-rep> <units> [--top N]
<units> normalises the instruction counts (e.g. chunk-warps = tasks * K).
"""
import csv
import collections
import io
import subprocess
import sys


def main():
    rep, units = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 60
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, agg, smp, src = None, collections.Counter(), collections.Counter(), {}
    per_file = collections.Counter()
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] == "Line No" or not r[0]:
            continue
        try:
            n, s = float(r[7]), float(r[4] or 0)
        except ValueError:
            continue
        key = (cur, int(r[0]))
        agg[key] += n
        smp[key] += s
        src[key] = r[1][:90]
        per_file[cur] += n
    tot, tots = sum(agg.values()), sum(smp.values()) or 1
    print("instructions per unit: %.1f" % (tot / units))
    for f, v in per_file.most_common():
        print("  %-28s %.1f" % (f, v / units))
    print("%-30s %8s %6s  %s" % ("line", "inst/u", "stall%", "source"))
    for k, v in agg.most_common(top):
        print("%-30s %8.1f %6.1f  %s" % ("%s:%d" % k, v / units, smp[k] / tots * 100, src[k]))


if __name__ == "__main__":
    main()
