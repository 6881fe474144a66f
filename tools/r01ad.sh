TAG=base python tools/layer_times.py 2>&1 | tail -2
for v in kas6 kas8 kas3; do FTC_LIB_PATH=build/variants/$v.so TAG=$v python tools/layer_times.py 2>&1 | tail -2; done
FTC_TC_B_STAGES=3 TAG=sb3 python tools/layer_times.py 2>&1 | tail -2
