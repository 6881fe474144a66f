# r02i: the r02h failures after the turn-barrier fence, determinism, the C++ programs
set -x
timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_cpp_api.py tests/test_gpu_gates.py tests/test_gpu_scale.py -m gpu -q -x --durations=10 > gpurun_out/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
DET_REPS=60 timeout 600 python tools/determinism.py > gpurun_out/r02i_det.log 2>&1; echo "det rc=$?"
