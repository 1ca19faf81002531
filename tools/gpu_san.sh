#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck
# (under gpurun, after tools/san_target.py exited 0 without the sanitizer).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TOOL:-memcheck}
timeout 200 python tools/san_target.py > gpurun_out/san_plain.txt 2>&1 && \
timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/san_target.py > gpurun_out/san_$T.txt 2>&1
echo "rc=$?" >> gpurun_out/san_$T.txt
