set -e
export N=256
LAYER=1024,256,14,1 python tools/one_fwd.py > gpurun_out/q1.log 2>&1
LAYER=256,1024,14,1 python tools/one_fwd.py > gpurun_out/q2.log 2>&1
LAYER=1024,256,14,1 ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_1x1_c1024 python tools/one_fwd.py > /dev/null 2>&1
LAYER=256,1024,14,1 ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 2 -c 1 -o gpurun_out/r02_1x1_c256 python tools/one_fwd.py > /dev/null 2>&1
