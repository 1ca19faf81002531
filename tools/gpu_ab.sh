#!/bin/bash
# under gpurun: kernel times of the in-tree library and of every ab/libvtrace_<tag>.so on the
# same box (interleaved twice), then an optional pytest selection on the in-tree library
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
P=gpurun_out/${TAG:-ab}
CFGS=${CFGS:-"large large:B=4096 large:B=2048 stress"}
: > ${P}_kt.txt
for rep in 1 2; do
  echo "== base (in-tree) rep $rep" >> ${P}_kt.txt
  timeout 300 python tools/kernel_time.py $CFGS --pdl >> ${P}_kt.txt 2>&1
  for so in ab/libvtrace_*.so; do
    echo "== $so rep $rep" >> ${P}_kt.txt
    KT_LIB=$so timeout 300 python tools/kernel_time.py $CFGS --pdl >> ${P}_kt.txt 2>&1
  done
done
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -q -x > ${P}_tests.txt 2>&1; echo "rc=$?" >> ${P}_tests.txt
fi
