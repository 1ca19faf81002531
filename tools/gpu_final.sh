#!/bin/bash
# under gpurun: the round pass (tools/gpu_round.sh) then one ncu --set full capture each of the
# large and stress column-block launches, exported as raw csv (traffic, warps active, throughput)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-fin} bash tools/gpu_round.sh
P=gpurun_out/${TAG:-fin}
for cfg in large stress; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'vtrace_' -s 5 -c 1 -o ${P}_full_$cfg python tools/ncu_target.py $cfg 6 0 > ${P}_full_$cfg.log 2>&1
  ncu -i ${P}_full_$cfg.ncu-rep --page raw --csv > ${P}_full_${cfg}_raw.csv 2>&1
  rm -f ${P}_full_$cfg.ncu-rep
done
