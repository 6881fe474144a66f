timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_gates.py -m gpu -q -x -k "c3_corpus or b3_proj or c8 or yolov2" > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
timeout 1200 python -m pytest tests/test_gpu_scale.py -m gpu -q -k "b3_proj or vgg19_b64_layers" > gpurun_out/r02e2_pytest.log 2>&1
