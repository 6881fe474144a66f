set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02w_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err; echo "bench rc=$?"
