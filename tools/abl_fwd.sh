#!/bin/bash
# Dev: forward ablation matrix for a few 1x1 layers (dev lib swapped in on the box)
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
for L in 1024,256,14,1 256,1024,14,1 2048,512,7,1 512,128,28,1; do
  for D in 0 256 128 384 1408 3456; do
    echo "#### LAYER=$L DBG=$D"
    LAYER=$L DBG=$D STAGES=0 python tools/fwd_trace.py 2>&1 | tail -3
  done
done
