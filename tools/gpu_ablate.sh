#!/bin/bash
# timing ablations of the column-task kernel (VTRACE_ABLATE builds; results are wrong by design)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-abl}
for A in ${ABLATIONS:-0 1 2 3 4 5}; do
  if [ "$A" = "0" ]; then python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  else VTRACE_ABLATE=$A python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1; fi
  timeout 300 python bench.py --config large --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > ${P}_$A.txt 2>&1
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
