"""Builds libvtrace.so (the C-ABI library) in-tree with nvcc for sm_100a.

Seven objects (the look-back kernel + the C ABI; the column-block kernels for bf16
and for fp32 logits; the learner update; the tcgen05 output layer; the learners' partials
sum over NVLink; the head fused with the path and its backward) are compiled in parallel
and linked into one shared library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libvtrace.so")
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, "vtrace_api.cu"), os.path.join(CSRC, "vtrace_cb_launch.cu"),
           os.path.join(CSRC, "learner_update.cu"), os.path.join(CSRC, "output_layer.cu"),
           os.path.join(CSRC, "partials_allreduce.cu"), os.path.join(CSRC, "head_fused.cu")]
# (source, object, defines): the column-block unit is compiled once per logits dtype
UNITS = [(SOURCES[0], "vtrace_api.o", []),
         (SOURCES[1], "vtrace_cb_bf16.o", ["-DVT_CB_PART=0"]),
         (SOURCES[1], "vtrace_cb_f32.o", ["-DVT_CB_PART=1"]),
         (SOURCES[2], "learner_update.o", []),
         (SOURCES[3], "output_layer.o", []),
         (SOURCES[4], "partials_allreduce.o", []),
         (SOURCES[5], "head_fused.o", [])]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                f"-I{os.path.join(ROOT, 'include')}", "-Xptxas", "-warn-spills"]


def _deps():
    return (SOURCES + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + [os.path.join(ROOT, "include", "vtrace.h")])


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in _deps())


def _extra_defines():
    extra = ["-DVTRACE_TIMING"] if os.environ.get("VTRACE_TIMING") else []
    for flag in ("VTRACE_SUM_F64",):  # A/B experiments only
        if os.environ.get(flag):
            extra.append("-D" + flag)
    if os.environ.get("VTRACE_ABLATE"):  # timing experiments only (wrong results)
        extra.append("-DVTRACE_ABLATE=" + os.environ["VTRACE_ABLATE"])
    # A/B experiments: extra -D flags, separated by commas (e.g. "VT_CT_NSTAGE=5,FOO")
    for d in filter(None, os.environ.get("VTRACE_DEFINES", "").split(",")):
        extra.append("-D" + d)
    return extra


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        extra = _extra_defines()
        objs, procs = [], []
        for src, oname, defs in UNITS:
            obj = os.path.join(CSRC, oname)
            cmd = [NVCC, *FLAGS, *extra, *defs, "-c", "-o", obj + ".tmp", src]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((subprocess.Popen(cmd), cmd))
            objs.append(obj)
        for p, cmd in procs:
            if p.wait() != 0:
                raise subprocess.CalledProcessError(p.returncode, cmd)
        for obj in objs:
            os.replace(obj + ".tmp", obj)
        link = [NVCC, *ARCH, "-shared", "-o", SO + ".tmp", *objs]
        if verbose:
            print(" ".join(link), file=sys.stderr)
        subprocess.check_call(link)
        os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
