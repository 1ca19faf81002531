#!/bin/bash
# default build: parity + margins + bench; then the no-arg-correction build: parity margins + bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-c9}
VTRACE_PARITY_REPORT=${P}_margin_def.jsonl timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_gpu_def.txt 2>&1; echo "rc=$?" >> ${P}_gpu_def.txt
for cfg in large stress; do timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > ${P}_bench_def_$cfg.txt 2>&1; done
VTRACE_NO_ARG_CORRECTION=1 python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_build_noarg.txt 2>&1
VTRACE_PARITY_REPORT=${P}_margin_noarg.jsonl timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "parity" > ${P}_gpu_noarg.txt 2>&1; echo "rc=$?" >> ${P}_gpu_noarg.txt
for cfg in large stress; do timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > ${P}_bench_noarg_$cfg.txt 2>&1; done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" >> ${P}_build_noarg.txt 2>&1
