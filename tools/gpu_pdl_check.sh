cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/pdl_tests.txt 2>&1; echo rc=$? >> gpurun_out/pdl_tests.txt
for a in "" "--no-overlap"; do timeout 300 python bench.py --steps 5000 --warmup 10 --no-cpu-baseline --no-e2e $a >> gpurun_out/pdl_bench.txt 2>&1; done
timeout 300 python bench.py --config stress --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/pdl_bench.txt 2>&1
