#!/bin/bash
# Dev: single-tap forward, lane-0 issue (DBG 8192) vs whole-warp issue (DBG 4096), plain and with the fused residual add
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
for L in 1024,256,14,1 256,1024,14,1 2048,512,7,1 512,2048,7,1 512,128,28,1 128,512,28,1 256,64,56,1 64,256,56,1 64,64,56,1; do
  for A in "" 1; do
  for D in 8192 4096; do
    echo -n "LAYER=$L ADD=$A DBG=$D : "
    ADD=$A LAYER=$L DBG=$D STAGES=0 python tools/fwd_trace.py 2>&1 | grep "CTA start"
  done
  done
done
