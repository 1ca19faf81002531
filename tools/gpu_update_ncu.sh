#!/bin/bash
# NEXT #4: update tests + bench, launch list, then one ncu --set full of the update kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-updn}
python -c "from paper_1802_01561_b200 import _build; _build.build()" > ${P}_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_rmsprop.py -q -p no:cacheprovider > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
for sz in deep shallow; do
  timeout 300 python bench.py --path update --update-size $sz --steps 2000 --warmup 10 > ${P}_bench_$sz.json 2> ${P}_bench_$sz.err
done
CMD="python bench.py --path update --steps 60 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > ${P}_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rmsprop --csv --log-file ${P}_launches.csv $CMD > ${P}_launch.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rmsprop -s 10 -c 1 -o ${P}_prof $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_ncu.log
