#!/bin/bash
# (under gpurun --gpus 2) timing build of the learners' update: per-call stamps, eager vs graph
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
VTRACE_DEFINES="RMS_TIMING" python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/rmsst_build.log 2>&1
for mode in replicated sharded; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 tools/rms_stamps.py $mode > gpurun_out/rmsst_$mode.txt 2>&1
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
grep -h "^{" gpurun_out/rmsst_*.txt
