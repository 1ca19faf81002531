#!/bin/bash
# (under gpurun --gpus 2) NEXT #4 at N = 2: the sharded update vs the replicated fused
# update vs NCCL, plus the one-GPU tests of the update
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-un2b}
timeout 600 python -m pytest tests/test_gpu_rmsprop.py -q -p no:cacheprovider > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
export VT_BENCH_WATCHDOG=250
for coll in symm_sharded symm nccl; do
  timeout 300 python bench.py --path update --update-collective $coll --update-size deep --gpus 2 --steps 2000 --warmup 10 --no-cpu-baseline > ${P}_$coll.json 2> ${P}_$coll.err
  echo "$coll rc=$?"
done
tail -3 ${P}_tests.txt
for coll in symm_sharded symm nccl; do grep -h "^{" ${P}_$coll.json | cut -c1-200; done
