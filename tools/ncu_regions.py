"""Per-source-region instruction/stall breakdown of an ncu report (dev tool)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, units = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


allrows = []
for si in starts:
    hdr = rows[si]
    ix = {}
    for j, h in enumerate(hdr):
        ix.setdefault(h, j)
    fname = rows[si - 2][1].split("/")[-1] if si >= 2 else ""
    for r in rows[si + 1:]:
        if not r or r[0] in ("Line No", "File Path", "Function Name"):
            break
        if len(r) == len(hdr) and r[0] != "":
            allrows.append((fname, int(r[0]), r[1], f(r[ix["Instructions Executed"]]),
                            f(r[ix["Warp Stall Sampling (All Samples)"]])))
src = open("paper_1802_01561_b200/csrc/vtrace_api.cu").read().splitlines()


def region(ln):
    for k in range(ln - 1, 0, -1):
        t = src[k - 1].strip()
        if t.startswith("// ----") or t.startswith("// ====") or t.startswith("template <"):
            return f"{k}:{t[:64]}"
    return "?"


tot = sum(x[3] for x in allrows)
samp = sum(x[4] for x in allrows) or 1
agg = defaultdict(lambda: [0, 0])
for fn, ln, txt, n, sm in allrows:
    key = region(ln) if fn == "vtrace_api.cu" else fn
    agg[key][0] += n
    agg[key][1] += sm
print(f"total warp-instr {tot:.0f}  per unit {tot / units:.0f}")
for k, (n, sm) in sorted(agg.items(), key=lambda x: -x[1][0])[:20]:
    print(f"{n / units:8.0f}/unit {n / tot * 100:5.1f}%  stall {sm / samp * 100:5.1f}%  {k}")
print("--- top lines")
for x in sorted(allrows, key=lambda x: -x[3])[:25]:
    print(f"{x[0][:12]:12s}{x[1]:>5} {x[3] / units:7.0f}/unit stall {x[4] / samp * 100:4.1f}%  {x[2][:80]}")
