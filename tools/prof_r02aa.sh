set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02aa_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02aa_pytest.log
DET_REPS=200 DET_SHAPE=16,64,56,64,3,1 timeout 300 python tools/det_diag.py > gpurun_out/r02aa_det64.log 2>&1
DET_REPS=200 timeout 300 python tools/det_diag.py > gpurun_out/r02aa_det512.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02aa_bench.json 2> gpurun_out/r02aa_bench.err; echo "bench rc=$?"
