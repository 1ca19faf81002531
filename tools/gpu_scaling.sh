#!/bin/bash
# (under gpurun --gpus 4) N = 1/2/4 bench lines: strong scaling with the NVLink partials
# sum (default) and with NCCL, weak scaling, and the driver's short form at N = 4.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export VT_BENCH_WATCHDOG=250
for n in 1 2 4; do timeout 300 python bench.py --gpus $n --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/s$n.json 2> gpurun_out/s$n.err; echo "s$n rc=$?"; done
for n in 2 4; do timeout 300 python bench.py --gpus $n --collective nccl --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/s${n}n.json 2> gpurun_out/s${n}n.err; echo "s${n}n rc=$?"; done
for n in 2 4; do timeout 300 python bench.py --gpus $n --weak --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/w$n.json 2> gpurun_out/w$n.err; echo "w$n rc=$?"; done
timeout 300 python bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/s4d.json 2> gpurun_out/s4d.err; echo "s4d rc=$?"
grep -h "^{" gpurun_out/s*.json gpurun_out/w*.json | cut -c1-250
for n in 2 4; do timeout 300 python bench.py --path update --gpus $n --steps 2000 --warmup 10 --no-cpu-baseline > gpurun_out/u$n.json 2> gpurun_out/u$n.err; echo "u$n rc=$?"; done
grep -h "^{" gpurun_out/u*.json | cut -c1-250
