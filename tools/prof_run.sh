export FTC_TC_DRAIN_CHUNKS=4
python tools/tc_time.py > gpurun_out/pre.log 2>&1 && python tools/conv_once.py alex >> gpurun_out/pre.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_conv_tc -s 3 -c 1 -o gpurun_out/prof_tc_nhwc_g4 python tools/conv_once.py alex > gpurun_out/ncu_nhwc.log 2>&1
