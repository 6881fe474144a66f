FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/r02ag_fault.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ag_fault_launches.csv env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/r02ag_fault_ncu.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02ag_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ag_pytest.log
