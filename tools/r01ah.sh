timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01ah_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01ah_pytest.log; tail -2 gpurun_out/r01ah_pytest.log
python tools/fault_times.py 2>&1 | grep -E "run|stage=(coc|rc|clc|fc|recompute)|clean"
