#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/${TAG:-tp}.txt
: > $O
for args in ${PROBES:-"4 8 4 0 16 0" "4 8 4 0 16 1" "4 8 4 0 16 2" "4 8 4 1 16 0" "4 8 4 1 16 1" "4 8 4 1 16 2" "8 8 4 0 8 1" "8 8 4 1 8 1" "12 8 4 1 4 1" "12 8 4 0 4 1"}; do
  timeout 60 ./tools/tma_probe ${args//_/ } >> $O 2>&1
done
