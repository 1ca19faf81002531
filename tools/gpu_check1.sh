#!/bin/bash
# first GPU call: probe MUFU accuracy, parity tests (both exp modes), a short bench
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi > gpurun_out/c1_nvsmi.txt 2>&1
timeout 120 ./tools/mufu_probe > gpurun_out/c1_mufu.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "full_size" > gpurun_out/c1_parity_f64.txt 2>&1
echo "rc=$?" >> gpurun_out/c1_parity_f64.txt
VTRACE_EXP_MODE=mufu timeout 600 python -m pytest tests -m gpu -q -k "full_size" > gpurun_out/c1_parity_mufu.txt 2>&1
echo "rc=$?" >> gpurun_out/c1_parity_mufu.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/c1_gpu_all.txt 2>&1
echo "rc=$?" >> gpurun_out/c1_gpu_all.txt
timeout 300 python bench.py --steps 2000 --warmup 10 --no-cpu-baseline > gpurun_out/c1_bench_f64.txt 2>&1
echo "rc=$?" >> gpurun_out/c1_bench_f64.txt
VTRACE_EXP_MODE=mufu timeout 300 python bench.py --steps 2000 --warmup 10 --no-cpu-baseline > gpurun_out/c1_bench_mufu.txt 2>&1
echo "rc=$?" >> gpurun_out/c1_bench_mufu.txt
