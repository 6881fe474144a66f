timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01x_pytest.log; tail -5 gpurun_out/r01x_pytest.log
timeout 300 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01x_c1.json 2> gpurun_out/r01x_c1.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01x_alex.json 2> gpurun_out/r01x_alex.err
python - <<'PY'
import json
for f in ("gpurun_out/r01x_alex.json","gpurun_out/r01x_c1.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], "ovh%", round(d["abft_overhead_pct"],2), "ms", d["ms_per_step"], "unprot", d["ms_per_step_unprotected"], "frac", round(d["roofline"]["frac"],3), "e2e", d["e2e"]["value"])
PY
