#!/bin/bash
# (under gpurun) the fused head: GPU tests, one bench line, a launch list
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-hf}
timeout 300 python -m pytest tests/test_gpu_head_fused.py -q -p no:cacheprovider > ${P}_tests.txt 2>&1
echo "rc=$?" >> ${P}_tests.txt
if grep -q "passed" ${P}_tests.txt && ! grep -q "failed" ${P}_tests.txt; then
  timeout 300 python bench.py --path head_fused --steps 50 --warmup 5 > ${P}_bench.json 2> ${P}_bench.err
  echo "bench rc=$?" >> ${P}_bench.err
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:head_ --csv --log-file ${P}_launches.csv python bench.py --path head_fused --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > ${P}_ncu.log 2>&1
fi
tail -4 ${P}_tests.txt; cat ${P}_bench.json 2>/dev/null | cut -c1-600
if [ -n "$FULL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:head_fused -s 3 -c 1 -o ${P}_prof python bench.py --path head_fused --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > ${P}_ncufull.log 2>&1
  echo "ncu rc=$?" >> ${P}_ncufull.log
fi
