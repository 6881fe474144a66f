timeout 900 python -m pytest tests -m gpu -x -q -k "host_pipeline" > gpurun_out/r01m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01m_pytest.log; tail -3 gpurun_out/r01m_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01m_alex.json 2> gpurun_out/r01m_alex.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r01m_alex.json").read().strip().splitlines()[-1])
print(d["value"], "ovh%", round(d["abft_overhead_pct"],2), "frac", round(d["roofline"]["frac"],3), "e2e", d["e2e"])
PY
