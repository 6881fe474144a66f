export SHAPES="16,64,56,64,3,1;64,64,224,64,3,1;64,256,56,256,3,1;64,512,28,512,3,1;128,96,27,256,5,2"
for v in base nosplit onecommit0; do
  L=""; [ $v != base ] && L=build/variants/$v.so
  FTC_LIB_PATH=$L timeout 600 python tools/shape_times.py > gpurun_out/r02ak_$v.log 2>&1
  FTC_LIB_PATH=$L timeout 600 python tools/layer_times.py | grep unprot >> gpurun_out/r02ak_$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_paths.py -m gpu -q -x > gpurun_out/r02ak_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ak_pytest.log
