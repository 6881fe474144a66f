set -x
timeout 600 python tools/layer_times.py > gpurun_out/r02r_times.log 2>&1
FTC_LIB_PATH=build/variants/g1.so timeout 600 python tools/layer_times.py > gpurun_out/r02r_times_g1.log 2>&1
timeout 300 python tools/tc_trace2.py > gpurun_out/r02r_trace.log 2>&1
DET_REPS=300 timeout 300 python tools/det_diag.py > gpurun_out/r02r_det.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_nets.py -m gpu -q -x > gpurun_out/r02r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_pytest.log
