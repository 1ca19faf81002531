#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-n2f}
python -c "from paper_1802_01561_b200 import _build; _build.build()" > ${P}_build.txt 2>&1
port=29700
for coll in symm nccl; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --path update --update-collective $coll --gpus 2 --steps 2000 --warmup 10 --no-cpu-baseline > ${P}_upd_${coll}.json 2> ${P}_upd_${coll}.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29710 bench.py --gpus 2 > ${P}_vtrace.json 2> ${P}_vtrace.err
