timeout 900 python -m pytest tests -m gpu -x -q -k "state or glue or net" > gpurun_out/r01ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01ab_pytest.log; tail -2 gpurun_out/r01ab_pytest.log
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01ab_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01ab_ncu.log 2>&1
python tools/launches_table.py gpurun_out/r01ab_launches.csv 3 | grep -E "cd1_parts"
