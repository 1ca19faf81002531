#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TAG:-t4}
VTRACE_TIMING=1 python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/${T}_build.txt 2>&1
for cfg in large stress; do timeout 300 python tools/phase_timing.py $cfg > gpurun_out/${T}_timing_$cfg.txt 2>&1; done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" >> gpurun_out/${T}_build.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_gpu.txt
for cfg in large stress; do timeout 300 python bench.py --config $cfg --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_$cfg.txt 2>&1; done
