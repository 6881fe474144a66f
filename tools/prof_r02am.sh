timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02am_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02am_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02am_bench.json 2> gpurun_out/r02am_bench.err
timeout 600 ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02am_resnet_launches.csv python bench.py --workload resnet18 --steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > /dev/null 2>&1
