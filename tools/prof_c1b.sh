python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1b_plain.json 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/c1b_launches.csv \
    python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1b_ncu.log 2>&1
FTC_NO_FUSED=1 ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/c1b_launches_nofused.csv \
    python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1b_ncu2.log 2>&1
echo done
