#!/bin/bash
# NEXT #4 at N = 2: fused symmetric-memory update vs NCCL all-reduce + update
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-un2}
python -c "from paper_1802_01561_b200 import _build; _build.build()" > ${P}_build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
port=29620
for coll in symm nccl; do
  for sz in deep shallow; do
    port=$((port+1))
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --path update --update-collective $coll --update-size $sz --gpus 2 --steps 2000 --warmup 10 --no-cpu-baseline > ${P}_${coll}_$sz.json 2> ${P}_${coll}_$sz.err
  done
done
