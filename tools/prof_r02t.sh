set -x
timeout 600 python tools/layer_times.py > gpurun_out/r02t_times.log 2>&1
timeout 300 python tools/tc_trace2.py > gpurun_out/r02t_trace.log 2>&1
