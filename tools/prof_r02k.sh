set -x
export DET_REPS=400
FTC_TC_DEBUG=8192 timeout 300 python tools/det_diag.py > gpurun_out/r02k_nock.log 2>&1
FTC_TC_DEBUG=4096 timeout 300 python tools/det_diag.py > gpurun_out/r02k_noatom.log 2>&1
FTC_TC_DEBUG=12288 timeout 300 python tools/det_diag.py > gpurun_out/r02k_none.log 2>&1
FTC_LIB_PATH=build/variants/noearly.so timeout 300 python tools/det_diag.py > gpurun_out/r02k_noearly.log 2>&1
FTC_LIB_PATH=build/variants/commit1.so timeout 300 python tools/det_diag.py > gpurun_out/r02k_commit1.log 2>&1
timeout 300 python tools/det_diag.py > gpurun_out/r02k_base.log 2>&1
