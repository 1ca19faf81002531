#!/bin/bash
# v2 kernel: parity both exp modes (with margins), bench 4 configs both modes, ncu on large (default mode)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-c3}
VTRACE_PARITY_REPORT=${P}_margin_mufu.jsonl timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_gpu_mufu.txt 2>&1; echo "rc=$?" >> ${P}_gpu_mufu.txt
VTRACE_EXP_MODE=f64 VTRACE_PARITY_REPORT=${P}_margin_f64.jsonl timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_gpu_f64.txt 2>&1; echo "rc=$?" >> ${P}_gpu_f64.txt
for cfg in large stress dmlab atari; do
  timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline > ${P}_bench_mufu_$cfg.txt 2>&1
  VTRACE_EXP_MODE=f64 timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > ${P}_bench_f64_$cfg.txt 2>&1
done
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > ${P}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vtrace_ -s 6 -c 1 -o ${P}_prof $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_ncu.log
