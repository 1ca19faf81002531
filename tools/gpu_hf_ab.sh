#!/bin/bash
# (under gpurun) A/B builds of the fused head: for each "tag:DEFINES", rebuild and time.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-hfab}.txt
: > $OUT
for v in "$@"; do
  tag=${v%%:*}; defs=${v#*:}
  VTRACE_DEFINES="$defs" python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/build_$tag.log 2>&1 || { echo "build $tag failed" >> $OUT; continue; }
  echo "== $tag ($defs)" >> $OUT
  timeout 300 python tools/hf_time.py ${CFGS:-100 8192 256 18} >> $OUT 2>&1
done
python -c "from paper_1802_01561_b200 import _build; _build.build(force=True)" > gpurun_out/rebuild.log 2>&1
cat $OUT
