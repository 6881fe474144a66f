# bench lines (AlexNet, config 1) + the timed-region launch list with per-launch DRAM bytes
set -e
python bench.py --no-cpu-baseline > gpurun_out/r01c_alex.json 2> gpurun_out/r01c_alex.err
python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01c_c1.json 2> gpurun_out/r01c_c1.err
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01c_launches_alex.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01c_ncu.log 2>&1
