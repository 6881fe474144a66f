timeout 900 python -m pytest tests -m gpu -x -q -k "backward or model_io or cli" > gpurun_out/r01l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01l_pytest.log; tail -25 gpurun_out/r01l_pytest.log
