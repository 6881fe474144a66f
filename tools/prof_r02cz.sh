set -x
timeout 300 python tools/tc_trace3.py > gpurun_out/r02cz_trace_c3.log 2>&1
TRACE_BITS=16384 timeout 300 python tools/tc_trace3.py > gpurun_out/r02cz_trace_c3_nostore.log 2>&1
SHAPES="64,64,112,128,3,1;64,128,112,128,3,1;64,256,56,256,3,1" timeout 300 python tools/shape_times.py > gpurun_out/r02cz_shapes.log 2>&1
FTC_TC_DEBUG=16384 SHAPES="64,64,112,128,3,1;64,128,112,128,3,1;64,256,56,256,3,1" timeout 300 python tools/shape_times.py > gpurun_out/r02cz_shapes_nostore.log 2>&1
echo done
