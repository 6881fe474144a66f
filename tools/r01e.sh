# fused clean path: GPU tests, smoke, bench (AlexNet + config1), launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01e_pytest.log
tail -30 gpurun_out/r01e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01e_smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01e_alex.json 2> gpurun_out/r01e_alex.err
timeout 300 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/r01e_c1.json 2> gpurun_out/r01e_c1.err
FTC_NO_FUSED=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r01e_alex_nofused.json 2> gpurun_out/r01e_alex_nofused.err
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r01e_launches_alex.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01e_ncu.log 2>&1
tail -2 gpurun_out/r01e_smoke.log; cat gpurun_out/r01e_alex.json gpurun_out/r01e_c1.json gpurun_out/r01e_alex_nofused.json; tail -5 gpurun_out/r01e_alex.err
