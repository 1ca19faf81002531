#!/bin/bash
# usage (under gpurun): TAG=x CFG=large bash tools/gpu_prof.sh
# GPU parity tests (no -x), then one plain run and the ncu full capture of the
# column-block kernel on $CFG.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-p}
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -q > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
fi
CMD="python tools/ncu_target.py ${CFG:-large} 6 ${KERN:-0}"
timeout 120 $CMD > ${P}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'vtrace_' -s 5 -c 1 -o ${P}_prof $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_ncu.log
