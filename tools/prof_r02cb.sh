set -x
timeout 600 python tools/c4_diag.py > gpurun_out/r02cb_diag.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor.sum,smsp__cycles_active.avg --clock-control none --csv -k regex:"k_conv_tc|k_nchw|k_nhwc" --log-file gpurun_out/r02cb_diag_ncu.csv python tools/c4_diag.py > gpurun_out/r02cb_diag_ncu.log 2>&1
echo done
