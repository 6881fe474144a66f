export SHAPES="16,64,56,64,3,1;64,64,224,64,3,1;256,64,56,64,3,1;64,32,208,64,3,1"
timeout 600 python tools/shape_times.py > gpurun_out/r02ao_f32.log 2>&1
FTC_LIB_PATH=build/variants/epi64.so timeout 600 python tools/shape_times.py > gpurun_out/r02ao_f64.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nets.py tests/test_gpu_scale.py tests/test_gpu_determinism.py -m gpu -q -x > gpurun_out/r02ao_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_pytest.log
