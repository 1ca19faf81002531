#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${TAG:-pdlab}.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "overlap or column_task or balanced or full_size" > gpurun_out/${TAG:-pdlab}_tests.txt 2>&1; echo rc=$? >> gpurun_out/${TAG:-pdlab}_tests.txt
for e in "VTRACE_CT_BALANCED=1" "VTRACE_CT_BALANCED=0"; do for a in "" "--no-overlap"; do
  echo "$e $a" >> $O
  env $e timeout 300 python bench.py --steps 5000 --warmup 10 --no-cpu-baseline --no-e2e $a >> $O 2>&1
done; done
