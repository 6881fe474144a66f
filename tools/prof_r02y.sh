export SHAPES="16,64,56,64,3,1;64,64,224,64,3,1;256,64,56,64,3,1"
FTC_LIB_PATH=build/variants/narrow3.so timeout 600 python tools/shape_times.py > gpurun_out/r02y_g3.log 2>&1
FTC_LIB_PATH=build/variants/narrow4.so timeout 600 python tools/shape_times.py > gpurun_out/r02y_g4.log 2>&1
