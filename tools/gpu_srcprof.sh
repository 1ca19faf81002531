#!/bin/bash
# under gpurun: baseline kernel times, then one ncu full capture of the large column-block
# kernel exported as the per-SASS source page (dynamic instruction counts per line)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-sp}
timeout 300 python tools/kernel_time.py large large:B=4096 large:B=2048 stress --pdl > ${P}_kt.txt 2>&1
CMD="python tools/ncu_target.py ${CFG:-large} 6 0"
timeout 120 $CMD > ${P}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'vtrace_' -s 5 -c 1 -o ${P}_prof $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_ncu.log
ncu -i ${P}_prof.ncu-rep --page source --csv --print-source sass > ${P}_source.csv 2>&1
ncu -i ${P}_prof.ncu-rep --page raw --csv > ${P}_raw.csv 2>&1
ls -la gpurun_out
