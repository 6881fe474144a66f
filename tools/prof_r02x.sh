timeout 600 python tools/shape_times.py > gpurun_out/r02x_g2.log 2>&1
FTC_LIB_PATH=build/variants/narrow1.so timeout 600 python tools/shape_times.py > gpurun_out/r02x_g1.log 2>&1
