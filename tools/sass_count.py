#!/usr/bin/env python
"""Static SASS census of one kernel of libvtrace.so (no GPU needed).

usage: python tools/sass_count.py <substring of mangled name> [--loop]
Prints the instruction count by opcode for the whole function or, with
--loop, for the largest backward-branch loop body (the per-chunk loop).
"""
import re
import subprocess
import sys
from collections import Counter

SO = "paper_1802_01561_b200/libvtrace.so"


def main():
    pat = sys.argv[1]
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    funcs = out.split("Function : ")
    fn = [f for f in funcs if f.split("\n", 1)[0].find(pat) >= 0]
    if not fn:
        sys.exit("no function matches " + pat)
    f = fn[0]
    print(f.split("\n", 1)[0])
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    lo, hi = 0, ins[-1][0]
    if "--loop" in sys.argv:
        best = None
        for addr, txt in ins:
            m = re.search(r"BRA\s.*?0x([0-9a-f]+)", txt)
            if m and int(m.group(1), 16) < addr:
                span = addr - int(m.group(1), 16)
                if best is None or span > best[1] - best[0]:
                    best = (int(m.group(1), 16), addr)
        lo, hi = best
    ops = Counter()
    for addr, txt in ins:
        if lo <= addr <= hi:
            toks = txt.split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            ops[op.split(".")[0]] += 1
    print("range 0x%x-0x%x: %d instructions" % (lo, hi, sum(ops.values())))
    for op, n in ops.most_common(40):
        print("  %-10s %d" % (op, n))


if __name__ == "__main__":
    main()
