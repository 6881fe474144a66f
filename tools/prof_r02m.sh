set -x
DET_REPS=400 timeout 300 python tools/det_diag.py > gpurun_out/r02m_det.log 2>&1
timeout 600 python tools/layer_times.py > gpurun_out/r02m_times.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_nets.py -m gpu -q -x > gpurun_out/r02m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02m_pytest.log
