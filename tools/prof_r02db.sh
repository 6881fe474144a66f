set -x
S="64,64,112,128,3,1;64,128,112,128,3,1;64,256,56,256,3,1;64,512,28,512,3,1;64,64,224,64,3,1"
SHAPES="$S" timeout 300 python tools/shape_times.py > gpurun_out/r02db_shapes_base.log 2>&1
for v in spin20 spin50 spin100; do
FTC_LIB_PATH=$PWD/build/variants/$v.so SHAPES="$S" timeout 300 python tools/shape_times.py > gpurun_out/r02db_shapes_$v.log 2>&1
done
FTC_LIB_PATH=$PWD/build/variants/spin50.so timeout 300 python tools/tc_trace3.py > gpurun_out/r02db_trace_spin50.log 2>&1
echo done
