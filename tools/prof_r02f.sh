python tools/determinism.py > gpurun_out/r02f_det.log 2>&1
FTC_NO_PDL=1 python tools/determinism.py > gpurun_out/r02f_det_nopdl.log 2>&1
FTC_LIB_PATH=build/variants/noearly.so python tools/determinism.py > gpurun_out/r02f_det_noearly.log 2>&1
