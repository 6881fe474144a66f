timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01p_pytest.log; tail -30 gpurun_out/r01p_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01p_alex.json 2> gpurun_out/r01p_alex.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r01p_alex.json").read().strip().splitlines()[-1])
print(d["value"], "ovh%", round(d["abft_overhead_pct"],2), "ms", d["ms_per_step"], "unprot", d["ms_per_step_unprotected"], "frac", round(d["roofline"]["frac"],3), "e2e", d["e2e"]["value"])
PY
