set -e
python tools/alex_convs.py > gpurun_out/plain_alex.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 20 -c 5 -o gpurun_out/prof_r01_alex_convs python tools/alex_convs.py > gpurun_out/ncu_alex.log 2>&1
