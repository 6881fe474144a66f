set -x
timeout 300 python tools/seq_time.py > gpurun_out/${PFX}_seq.log 2>&1
FTC_SEQ_STAGED=0 timeout 300 python tools/seq_time.py > gpurun_out/${PFX}_seq_old.log 2>&1
FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/${PFX}_fault.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${PFX}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${PFX}_pytest.log
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M --log-file gpurun_out/${PFX}_fault_launches.csv env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/${PFX}_fault_ncu.log 2>&1
echo done
