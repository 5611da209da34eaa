# list the kernels of the library with register spills (ptxas -v)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v \
  -o /tmp/spills_check.so "$(dirname "$0")/../paper_1808_05567_b200/csrc/dconv_capi.cu" 2>&1 | \
  awk '/Function properties for/{f=$NF} /spill stores/{ if ($5 != "0" || $9 != "0") print f, $0 }'
