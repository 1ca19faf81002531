#!/bin/bash
# Round-style GPU pass (under gpurun): build + smoke, the GPU tests, the default bench line
# (and the driver's short form), the reference arm, the other configs, the update and head
# paths, then the ncu launch list of a short bench run (one ncu tool per call).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-rd}
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1; echo "rc=$?" >> ${P}_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_gpu_tests.txt 2>&1; echo "rc=$?" >> ${P}_gpu_tests.txt
timeout 600 python bench.py > ${P}_bench.json 2> ${P}_bench.err; echo "rc=$?" >> ${P}_bench.err
timeout 600 python bench.py --steps 20 --warmup 3 > ${P}_bench_driver_form.json 2>> ${P}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > ${P}_bench_ref.json 2> ${P}_bench_ref.err; echo "rc=$?" >> ${P}_bench_ref.err
for cfg in atari dmlab stress toy; do timeout 300 python bench.py --config $cfg --no-cpu-baseline > ${P}_bench_$cfg.json 2>> ${P}_bench.err; done
timeout 300 python bench.py --path update > ${P}_bench_update.json 2>> ${P}_bench.err
timeout 300 python bench.py --path head --steps 200 --warmup 5 > ${P}_bench_head.json 2>> ${P}_bench.err
timeout 300 python bench.py --path head_fused --steps 100 --warmup 5 > ${P}_bench_head_fused.json 2>> ${P}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vtrace_ -c 200 --csv --log-file ${P}_launches.csv python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_launches.log 2>&1; echo "rc=$?" >> ${P}_launches.log
