mkdir -p gpurun_out
export VT_BENCH_WATCHDOG=250
for n in 1 2 4; do timeout 300 python bench.py --gpus $n --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/s$n.json 2> gpurun_out/s$n.err; echo "s$n rc=$?"; done
for n in 2 4; do timeout 300 python bench.py --gpus $n --weak --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/w$n.json 2> gpurun_out/w$n.err; echo "w$n rc=$?"; done
timeout 300 python bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/s4d.json 2> gpurun_out/s4d.err; echo "s4d rc=$?"
grep -h "^{" gpurun_out/s*.json gpurun_out/w*.json | cut -c1-250
