set -x
timeout 600 python tools/layer_times.py > gpurun_out/r02n_base.log 2>&1
FTC_TC_DEBUG=8 timeout 600 python tools/layer_times.py > gpurun_out/r02n_nomma.log 2>&1
FTC_TC_DEBUG=4 timeout 600 python tools/layer_times.py > gpurun_out/r02n_nodrain.log 2>&1
FTC_TC_DEBUG=12 timeout 600 python tools/layer_times.py > gpurun_out/r02n_nomma_nodrain.log 2>&1
FTC_TC_DEBUG=1 timeout 600 python tools/layer_times.py > gpurun_out/r02n_noA.log 2>&1
FTC_TC_DEBUG=2 timeout 600 python tools/layer_times.py > gpurun_out/r02n_noAst.log 2>&1
FTC_LIB_PATH=build/variants/order1.so timeout 600 python tools/layer_times.py > gpurun_out/r02n_order1.log 2>&1
