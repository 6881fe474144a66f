# r01e profiles: fused clean path (Co5 in the conv, glue Cd1) -- launch list of the timed
# region with DRAM bytes, ncu --set full of the 5 convs and of the glue/Cd1/detect kernels
set -e
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01e2_plain.json 2> gpurun_out/r01e2_plain.err
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01e2_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01e2_ncu.log 2>&1
python tools/alex_convs.py > gpurun_out/r01e2_alex.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 20 -c 5 -o gpurun_out/r01e2_convs python tools/alex_convs.py > gpurun_out/r01e2_ncu_convs.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_act_pool|k_cd1_parts|k_detect_fused" -s 40 -c 11 -o gpurun_out/r01e2_aux python tools/alex_convs.py > gpurun_out/r01e2_ncu_aux.log 2>&1
echo done
