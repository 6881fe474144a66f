# r02b: full GPU suite (incl. BASELINE-scale parity), headline bench (VGG-19 b64 + extras), reference arm
set -x
timeout 1800 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err; echo "ref rc=$?"
