#!/bin/bash
# A/B build variants: for each VAR in $VARIANTS (env flag names, "base" = none):
# parity margins (full-size configs + params) and the large/stress bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-ab}
for V in ${VARIANTS:-base}; do
  if [ "$V" = "base" ]; then python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_${V}_build.txt 2>&1
  elif [[ "$V" == *=* ]]; then env $V python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_${V}_build.txt 2>&1
  else env $V=1 python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_${V}_build.txt 2>&1; fi
  VTRACE_PARITY_REPORT=${P}_${V}_margin.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "full_size or params or column_task" > ${P}_${V}_gpu.txt 2>&1; echo "rc=$?" >> ${P}_${V}_gpu.txt
  for cfg in large stress; do timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > ${P}_${V}_bench_$cfg.txt 2>&1; done
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
