#!/bin/bash
# (under gpurun --gpus 2) bench.py --path update at N = 2 with the RMS_TIMING build: the
# per-call stamps of its timed (graph) region, replicated and sharded
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
VTRACE_DEFINES="RMS_TIMING" python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/rmsbs_build.log 2>&1
for coll in symm; do
  VT_RMS_STAMPS=1 timeout 300 python bench.py --path update --update-collective $coll --gpus 2 --steps 2000 --warmup 10 --no-cpu-baseline > gpurun_out/rmsbs_$coll.json 2> gpurun_out/rmsbs_$coll.err
  echo "== $coll"; grep -h '"rank"' gpurun_out/rmsbs_$coll.err; grep -h "^{" gpurun_out/rmsbs_$coll.json | cut -c1-200
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
