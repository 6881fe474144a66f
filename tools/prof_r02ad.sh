FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/r02ad_fault.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ad_fault_launches.csv env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/r02ad_fault_ncu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_nets.py tests/test_gpu_gates.py -m gpu -q -x > gpurun_out/r02ad_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ad_pytest.log
