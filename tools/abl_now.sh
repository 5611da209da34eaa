#!/bin/bash
# Dev: register-epilogue ablations (dev lib swapped in on the box)
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
for L in 64,64,56,3 512,512,7,3; do
  for D in 0 1 2 3 64 1024; do
    echo "#### LAYER=$L DBG=$D"
    LAYER=$L DBG=$D STAGES=0 python tools/fwd_trace.py 2>&1 | tail -3 | head -2
  done
done
