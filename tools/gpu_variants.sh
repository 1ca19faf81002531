#!/bin/bash
# A/B of compile-time variants (under gpurun): for each "tag:DEFINES" argument, rebuild
# libvtrace.so with VTRACE_DEFINES=DEFINES, time the configs in $CFGS ($KT_ARGS) and, with
# $TESTSEL set, run that pytest -k selection of the GPU parity tests.  The last variant's
# build stays in place; rebuild the default before other work.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-var}.txt
: > $OUT
for v in "$@"; do
  tag=${v%%:*}; defs=${v#*:}
  VTRACE_DEFINES="$defs" python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/build_$tag.log 2>&1 || { echo "build $tag failed" >> $OUT; continue; }
  echo "== $tag ($defs)" >> $OUT
  python tools/kernel_time.py ${CFGS:-large} $KT_ARGS >> $OUT 2>&1
  if [ -n "$TESTSEL" ]; then
    timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$TESTSEL" 2>&1 | tail -4 >> $OUT
  fi
done
