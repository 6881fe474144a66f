for e in "" "FTC_CO5_IN=1"; do
  env $e timeout 600 python bench.py --workload config1 --steps 20 --warmup 5 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/r02ap_c1_${e:-base}.json 2>/dev/null
done
env FTC_CO5_IN=1 timeout 600 ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ap_c1in_launches.csv python bench.py --workload config1 --steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > /dev/null 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ap_c1_launches.csv python bench.py --workload config1 --steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > /dev/null 2>&1
FTC_CO5_IN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k config1 > gpurun_out/r02ap_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ap_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_gates.py -m gpu -q -x >> gpurun_out/r02ap_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ap_pytest.log
