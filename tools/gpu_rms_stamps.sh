#!/bin/bash
# (under gpurun --gpus 2) timing build of the learners' update: per-call stamps and the host
# time of each graph replay, cooperative vs plain launch
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
port=29675
for defs in "RMS_TIMING" "RMS_TIMING,RMS_NO_COOP"; do
  VTRACE_DEFINES="$defs" python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/rmsst_build.log 2>&1
  port=$((port+1))
  echo "== $defs"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port tools/rms_stamps.py replicated 27 2>&1 | grep "^{"
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
