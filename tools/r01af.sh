timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01af_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01af_pytest.log; tail -2 gpurun_out/r01af_pytest.log
for w in resnet18 alexnet; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01af_$w.json 2> gpurun_out/r01af_$w.err
done
python - <<'PY'
import json
for w in ("resnet18","alexnet"):
    d=json.loads(open(f"gpurun_out/r01af_{w}.json").read().strip().splitlines()[-1])
    print(w, round(d["value"],1), "ovh%", round(d["abft_overhead_pct"],2), "ms", round(d["ms_per_step"],3), "unprot", round(d["ms_per_step_unprotected"],3), "frac", round(d["roofline"]["frac"],3), "det", d["detections_in_timed_region"])
PY
