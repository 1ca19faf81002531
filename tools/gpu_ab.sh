#!/bin/bash
# A/B variants: for each VAR in $VARIANTS ("base" = none; NAME=value or NAME -> NAME=1),
# the variable is set for the build, the parity-margin run and the large/stress bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-ab}
for V in ${VARIANTS:-base}; do
  if [ "$V" = "base" ]; then E="VTRACE_AB_BASE=1"; elif [[ "$V" == *=* ]]; then E="$V"; else E="$V=1"; fi
  env $E python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_${V}_build.txt 2>&1
  env $E VTRACE_PARITY_REPORT=${P}_${V}_margin.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "${PYTEST_K:-full_size or params or column_task}" > ${P}_${V}_gpu.txt 2>&1; echo "rc=$?" >> ${P}_${V}_gpu.txt
  for cfg in ${CONFIGS:-large stress}; do env $E timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > ${P}_${V}_bench_$cfg.txt 2>&1; done
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
