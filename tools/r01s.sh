timeout 900 python -m pytest tests -m gpu -x -q -k "glue or net or pipeline" > gpurun_out/r01s5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01s5_pytest.log; tail -3 gpurun_out/r01s5_pytest.log
python tools/glue_bench.py > gpurun_out/r01s5_glue.log 2>&1; grep "v2+ws" gpurun_out/r01s5_glue.log
TAG=cur python tools/layer_times.py 2>&1 | tail -2
