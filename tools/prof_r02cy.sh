set -x
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
B="--steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0"
timeout 900 ncu --nvtx --nvtx-include "timed_step/" $M --log-file gpurun_out/${PFX}_launches_vgg19.csv python bench.py --workload vgg19 $B > gpurun_out/${PFX}_ncu_vgg19.log 2>&1
echo done
