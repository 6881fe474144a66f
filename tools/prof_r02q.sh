TRACE_SHAPE=128,96,27,256,5,2 timeout 300 python tools/tc_trace2.py > gpurun_out/r02q_trace.log 2>&1; TRACE_BITS=8 timeout 300 python tools/tc_trace2.py > gpurun_out/r02q_trace_nomma.log 2>&1
