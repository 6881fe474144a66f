# re-validation after container re-creation: GPU tests, smoke, both bench workloads
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01d_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01d_smoke.log
timeout 600 python bench.py > gpurun_out/r01d_alex.json 2> gpurun_out/r01d_alex.err
timeout 300 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01d_c1.json 2> gpurun_out/r01d_c1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01d_ref.json 2> gpurun_out/r01d_ref.err
tail -3 gpurun_out/r01d_pytest.log; tail -2 gpurun_out/r01d_smoke.log; cat gpurun_out/r01d_alex.json gpurun_out/r01d_c1.json gpurun_out/r01d_ref.json
