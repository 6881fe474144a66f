TAG=lazy64 python tools/layer_times.py 2>&1 | tail -2
for v in lazy32 lazy128 lazy0; do FTC_LIB_PATH=build/variants/$v.so TAG=$v python tools/layer_times.py 2>&1 | tail -2; done
