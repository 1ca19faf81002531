#!/usr/bin/env python
"""A/B variant libraries (dev tool): recompiles the column-block units with extra
-D flags and links it with the other in-tree objects into ab/libvtrace_<tag>.so.

usage: python tools/ab_build.py <tag> [DEF[=V] ...] [-nvcc-flag ...]     (run the in-tree build first)
tools/kernel_time.py loads a variant with KT_LIB=ab/libvtrace_<tag>.so.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_01561_b200 import _build as b  # noqa: E402

tag = sys.argv[1]
defs = [a for a in sys.argv[2:] if not a.startswith("-")]
raw = [a for a in sys.argv[2:] if a.startswith("-")]  # extra nvcc flags as given
out = os.path.join(b.ROOT, "ab")
os.makedirs(out, exist_ok=True)
# both column-block units (bf16 holds the host plan, fp32 the other kernels), in parallel
new = {}
procs = []
for part, name in ((0, "vtrace_cb_bf16.o"), (1, "vtrace_cb_f32.o")):
    new[name] = os.path.join(out, f"{tag}_{name}")
    procs.append(subprocess.Popen([b.NVCC, *b.FLAGS, f"-DVT_CB_PART={part}", *["-D" + d for d in defs], *raw,
                                   "-c", "-o", new[name], b.SOURCES[1]]))
if any(p.wait() != 0 for p in procs):
    sys.exit("compile failed")
objs = [new.get(o, os.path.join(b.CSRC, o)) for _, o, _ in b.UNITS]
so = os.path.join(out, f"libvtrace_{tag}.so")
subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-o", so, *objs])
print(so)
