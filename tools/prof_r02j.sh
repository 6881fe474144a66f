set -x
DET_REPS=300 timeout 600 python tools/det_diag.py > gpurun_out/r02j_diag_prot.log 2>&1
DET_REPS=300 DET_MODE=conv timeout 600 python tools/det_diag.py > gpurun_out/r02j_diag_conv.log 2>&1
FTC_NO_PDL=1 DET_REPS=300 timeout 600 python tools/det_diag.py > gpurun_out/r02j_diag_nopdl.log 2>&1
DET_SHAPE=256,128,28,256,1,0 DET_REPS=200 timeout 600 python tools/det_diag.py > gpurun_out/r02j_diag_proj.log 2>&1
