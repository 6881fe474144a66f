# r01b profiles (final kernels of the round): bench lines, the timed-region launch list
# with DRAM bytes, ncu --set full of the 5 convs and of the glue / Cd1 / CoC-D kernels
set -e
python bench.py > gpurun_out/r01b_alex.json 2> gpurun_out/r01b_alex.err
python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01b_c1.json 2> gpurun_out/r01b_c1.err
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01b_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01b_ncu.log 2>&1
python tools/alex_convs.py > gpurun_out/r01b_alexconvs.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 20 -c 5 -o gpurun_out/r01b_convs python tools/alex_convs.py > gpurun_out/r01b_ncu_convs.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_act_pool|k_cd1_parts|k_detect_fused" -s 40 -c 11 -o gpurun_out/r01b_aux python tools/alex_convs.py > gpurun_out/r01b_ncu_aux.log 2>&1
echo done
