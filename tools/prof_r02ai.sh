ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r02ai_c1_launches.csv \
    python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/r02ai_ncu_c1.log 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r02ai_vgg_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/r02ai_ncu_vgg.log 2>&1
