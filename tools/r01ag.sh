timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r01ag_alex.json 2> gpurun_out/r01ag_alex.err; echo rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r01ag_alex.json").read().strip().splitlines()[-1])
print(d["value"], d["abft_overhead_pct"], d["faulted_forward"], d["config"]["tau_per_layer"])
PY
tail -3 gpurun_out/r01ag_alex.err
