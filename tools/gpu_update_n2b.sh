#!/bin/bash
# (under gpurun --gpus 2) NEXT #4 at N = 2: push / pull (replicated) / sharded / NCCL, plus the
# one-GPU tests of the update
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-un2b}
timeout 600 python -m pytest tests/test_gpu_rmsprop.py -q -p no:cacheprovider > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
export VT_BENCH_WATCHDOG=250
for coll in symm_push symm symm_sharded nccl; do
  timeout 300 python bench.py --path update --update-collective $coll --update-size deep --gpus ${NG:-2} --steps 2000 --warmup 10 --no-cpu-baseline > ${P}_$coll.json 2> ${P}_$coll.err
  echo "$coll rc=$?"
done
tail -3 ${P}_tests.txt
for coll in symm_push symm symm_sharded nccl; do python -c "
import json
for l in open('${P}_$coll.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$coll', {k: round(v*1000,2) for k,v in d.items() if k.endswith('ms_per_step')}, d.get('replicas_bitwise_equal'))
"; done
