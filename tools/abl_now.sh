#!/bin/bash
# Dev: role counters of the fused (residual add) 1x1 forwards and the 28x28 3x3 (dev lib swapped in on the box)
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
for L in 64,256,56,1 128,512,28,1 256,1024,14,1 512,2048,7,1; do
  for D in 0 512 1024 3456; do
    echo "#### ADD LAYER=$L DBG=$D"
    ADD=1 LAYER=$L DBG=$D STAGES=0 python tools/fwd_trace.py 2>&1 | tail -3 | head -2
  done
done
for L in 128,128,28,3; do
  for D in 0 1024 3456; do
    echo "#### LAYER=$L DBG=$D"
    LAYER=$L DBG=$D STAGES=0 python tools/fwd_trace.py 2>&1 | tail -3 | head -2
  done
done
