FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/r02af_fault.log 2>&1
timeout 300 python tools/seq_time.py > gpurun_out/r02af_seq.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_nets.py tests/test_gpu_gates.py tests/test_gpu_cpp_api.py -m gpu -q -x > gpurun_out/r02af_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02af_pytest.log
