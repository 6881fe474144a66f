timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01ac_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01ac_pytest.log; tail -15 gpurun_out/r01ac_pytest.log
