timeout 900 python -m pytest tests -m gpu -x -q -k "config1 or parity or state or fused" > gpurun_out/r01y_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01y_pytest.log; tail -2 gpurun_out/r01y_pytest.log
timeout 300 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01y_c1.json 2> gpurun_out/r01y_c1.err
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01y_c1_launches.csv \
    python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01y_ncu.log 2>&1
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r01y_c1.json").read().strip().splitlines()[-1])
print(d["value"], "ovh%", round(d["abft_overhead_pct"],2), "ms", d["ms_per_step"], "unprot", d["ms_per_step_unprotected"], "frac", round(d["roofline"]["frac"],3))
PY
python tools/launches_table.py gpurun_out/r01y_c1_launches.csv 3
