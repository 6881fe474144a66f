ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01z_resnet_launches.csv \
    python bench.py --workload resnet18 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r01z_ncu.log 2>&1
python tools/launches_table.py gpurun_out/r01z_resnet_launches.csv 1
