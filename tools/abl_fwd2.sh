#!/bin/bash
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
for D in 7552 4096; do
  echo "#### DBG=$D"
  LAYER=1024,256,14,1 DBG=$D STAGES=36 python tools/fwd_trace.py 2>&1 | tail -40
done
