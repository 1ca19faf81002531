#!/bin/bash
# one plain run then the ncu full capture of the large fused kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-n1}
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 300 $CMD > ${P}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^vtrace_(ct|ctb|fused)_kernel' -s 6 -c 1 -o ${P}_prof $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_ncu.log
