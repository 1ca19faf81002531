#!/usr/bin/env python
"""A/B variant libraries (dev tool): recompiles only the bf16 column-block unit with extra
-D flags and links it with the other in-tree objects into ab/libvtrace_<tag>.so.

usage: python tools/ab_build.py <tag> [DEF[=V] ...]     (run the in-tree build first)
tools/kernel_time.py loads a variant with KT_LIB=ab/libvtrace_<tag>.so.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_01561_b200 import _build as b  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "ab")
os.makedirs(out, exist_ok=True)
obj = os.path.join(out, f"cb_bf16_{tag}.o")
subprocess.check_call([b.NVCC, *b.FLAGS, "-DVT_CB_PART=0", *["-D" + d for d in defs], "-c", "-o", obj,
                       b.SOURCES[1]])
objs = [os.path.join(b.CSRC, o) for _, o, _ in b.UNITS if o != "vtrace_cb_bf16.o"] + [obj]
so = os.path.join(out, f"libvtrace_{tag}.so")
subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-o", so, *objs])
print(so)
