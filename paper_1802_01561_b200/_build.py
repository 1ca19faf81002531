"""Builds libvtrace.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libvtrace.so")
SOURCES = [os.path.join(HERE, "csrc", "vtrace_api.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", "vtrace_kernels.cuh"),
                  os.path.join(HERE, "csrc", "vtrace_ct.cuh"),
                  os.path.join(ROOT, "include", "vtrace.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", f"-I{os.path.join(ROOT, 'include')}",
         "-Xptxas", "-warn-spills"]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        extra = ["-DVTRACE_TIMING"] if os.environ.get("VTRACE_TIMING") else []
        for flag in ("VTRACE_SUM_F64",):  # A/B experiments only
            if os.environ.get(flag):
                extra.append("-D" + flag)
        if os.environ.get("VTRACE_ABLATE"):  # timing experiments only (wrong results)
            extra.append("-DVTRACE_ABLATE=" + os.environ["VTRACE_ABLATE"])
        cmd = [NVCC, *FLAGS, *extra, "-o", SO + ".tmp", *SOURCES]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
