#!/bin/bash
# (under gpurun) first GPU runs of the fused head; then the parity suite under the plain-sum
# build with the margin report.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_head_fused.py -q -x -p no:cacheprovider > gpurun_out/hf_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/hf_tests.txt
timeout 120 python -m pytest tests/test_gpu_output_layer.py tests/test_gpu_partials_allreduce.py -q -p no:cacheprovider > gpurun_out/ol_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/ol_tests.txt
VTRACE_PARITY_REPORT=$PWD/gpurun_out/margins_base.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/par_base.txt 2>&1
echo "rc=$?" >> gpurun_out/par_base.txt
VTRACE_DEFINES="CB_PLAIN_SUMS=1,CB_TD32=1" python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/build_ps.log 2>&1
VTRACE_PARITY_REPORT=$PWD/gpurun_out/margins_ps.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/par_ps.txt 2>&1
echo "rc=$?" >> gpurun_out/par_ps.txt
tail -5 gpurun_out/hf_tests.txt gpurun_out/ol_tests.txt gpurun_out/par_base.txt gpurun_out/par_ps.txt
