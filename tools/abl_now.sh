#!/bin/bash
# Dev: whole-warp single-tap issue loop forced on (4096) / off (8192) across the stack (dev lib swapped in on the box)
cp tools/devlib/libdconv_b200.so paper_1808_05567_b200/lib/libdconv_b200.so
export DCONV_DEV=1
for D in 0 4096 8192; do
  echo "#### DBG=$D"
  DBG=$D python tools/stack_profile.py 2>&1 | awk 'NR==1 || !seen[$2" "$3" "$4" "$5" "$6]++'
done
