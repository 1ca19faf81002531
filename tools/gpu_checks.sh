#!/bin/bash
# Device-side bounds checks (compute-sanitizer is closed on the pool): rebuild with
# -DVT_DEBUG_CHECKS (asserts on every shared-memory tile / stage / record index), run
# the small-launch target and the GPU parity tests on it, then restore the normal build.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-chk}
VTRACE_DEFINES=VT_DEBUG_CHECKS python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > ${P}_build.log 2>&1
timeout 300 python tools/san_target.py > ${P}_target.txt 2>&1; echo "rc=$?" >> ${P}_target.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" >> ${P}_build.log 2>&1
