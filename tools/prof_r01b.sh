set -e
python bench.py --steps 3 --warmup 3 > gpurun_out/plain_bench.log 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_timed.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
