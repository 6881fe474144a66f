timeout 300 python tools/tc_trace2.py > gpurun_out/r02s_trace.log 2>&1; TRACE_BITS=8 timeout 300 python tools/tc_trace2.py > gpurun_out/r02s_trace_nomma.log 2>&1
