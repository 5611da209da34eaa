#!/bin/bash
# Dev: bf16 weight-update ablations (dev lib swapped in on the box)
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
LAYERS="256,1024,14,1 1024,256,14,1 512,2048,7,1 256,256,14,3 64,64,56,3 512,512,7,3" python tools/upd3_ablate.py
