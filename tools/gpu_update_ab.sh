#!/bin/bash
# A/B of the learner-update kernel: VARIANTS of VTRACE_DEFINES, bench --path update
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-uab}
for V in ${VARIANTS:-base}; do
  if [ "$V" = "base" ]; then E="VTRACE_AB_BASE=1"; else E="VTRACE_DEFINES=$V"; fi
  env $E python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_${V}_build.txt 2>&1
  for sz in ${SIZES:-deep}; do
    env $E timeout 300 python bench.py --path update --update-size $sz --steps 3000 --warmup 10 --no-e2e --no-cpu-baseline > ${P}_${V}_$sz.json 2> ${P}_${V}_$sz.err
  done
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
