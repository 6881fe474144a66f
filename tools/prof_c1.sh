set -e
python bench.py --workload config1 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/plain_c1.log 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_timed.csv python bench.py --workload config1 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_c1.log 2>&1
