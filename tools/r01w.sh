for w in vgg19 resnet18 yolov2; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01w_$w.json 2> gpurun_out/r01w_$w.err; echo "$w rc=$?"
done
python - <<'PY'
import json
for w in ("vgg19","resnet18","yolov2"):
    try:
        d=json.loads(open(f"gpurun_out/r01w_{w}.json").read().strip().splitlines()[-1])
        print(w, round(d["value"],1), "ovh%", round(d["abft_overhead_pct"],2), "ms", round(d["ms_per_step"],3), "unprot", round(d["ms_per_step_unprotected"],3), "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],1), "det", d["detections_in_timed_region"])
    except Exception as e: print(w, "ERR", e)
PY
python - <<'PY'
import torch, time
x = torch.empty(79148544 // 4, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): y.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 79 MB pinned: {ms:.3f} ms = {79148544/ms/1e6:.1f} GB/s")
PY
tail -3 gpurun_out/r01w_*.err
