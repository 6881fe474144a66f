FTC_LIB_PATH=build/variants/order1.so timeout 600 python tools/layer_times.py > gpurun_out/r02v_o1.log 2>&1
FTC_LIB_PATH=build/variants/order2.so timeout 600 python tools/layer_times.py > gpurun_out/r02v_o2.log 2>&1
timeout 600 python tools/layer_times.py > gpurun_out/r02v_o0.log 2>&1
