set -x
export DET_REPS=500
FTC_LIB_PATH=build/variants/oneiss.so timeout 300 python tools/det_diag.py > gpurun_out/r02l_oneiss.log 2>&1
FTC_LIB_PATH=build/variants/oneiss.so DET_SHAPE=256,128,28,256,1,0 timeout 300 python tools/det_diag.py > gpurun_out/r02l_oneiss_proj.log 2>&1
timeout 300 python tools/det_diag.py > gpurun_out/r02l_base.log 2>&1
FTC_LIB_PATH=build/variants/oneiss.so timeout 600 python tools/layer_times.py > gpurun_out/r02l_oneiss_times.log 2>&1
timeout 600 python tools/layer_times.py > gpurun_out/r02l_base_times.log 2>&1
