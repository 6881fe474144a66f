timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01n_pytest.log; tail -3 gpurun_out/r01n_pytest.log
python tools/glue_bench.py > gpurun_out/r01n_glue.log 2>&1
for v in "base:" "nofused:FTC_NO_FUSED=1"; do
  tag=${v%%:*}; e=${v#*:}
  env TAG=$tag $e python tools/layer_times.py >> gpurun_out/r01n_layers.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01n_alex.json 2> gpurun_out/r01n_alex.err
timeout 300 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01n_c1.json 2> gpurun_out/r01n_c1.err
cat gpurun_out/r01n_glue.log gpurun_out/r01n_layers.log
python - <<'PY'
import json
for f in ("gpurun_out/r01n_alex.json","gpurun_out/r01n_c1.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], "ovh%", round(d["abft_overhead_pct"],2), "ms", d["ms_per_step"], "unprot", d["ms_per_step_unprotected"], "frac", round(d["roofline"]["frac"],3), "e2e", d["e2e"]["value"], "launches", d["launches_per_step"])
    except Exception as e: print(f, e)
PY
