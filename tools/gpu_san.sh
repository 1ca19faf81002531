#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --show-backtrace device --print-limit 5 python tools/repro_small.py dmlab loss 64 > gpurun_out/san_dmlab_loss.txt 2>&1
timeout 120 python tools/repro_small.py dmlab from 64 > gpurun_out/san_dmlab_from_plain.txt 2>&1
timeout 120 python tools/repro_small.py large loss 64 > gpurun_out/san_large_loss_plain.txt 2>&1
