#!/bin/bash
# NEXT #4 (learner update): parity tests, the full GPU suite, update bench lines
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-upd}
python -c "from paper_1802_01561_b200 import _build; _build.build()" > ${P}_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_rmsprop.py -q -p no:cacheprovider > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > ${P}_gpu_all.txt 2>&1; echo "rc=$?" >> ${P}_gpu_all.txt
for sz in deep shallow; do
  timeout 300 python bench.py --path update --update-size $sz --steps 2000 --warmup 10 > ${P}_bench_$sz.json 2> ${P}_bench_$sz.err
done
