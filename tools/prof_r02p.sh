set -x
for d in 0 31 24 28; do
FTC_LIB_PATH=build/variants/spin.so FTC_TC_DEBUG=$d timeout 600 python tools/layer_times.py > gpurun_out/r02p_spin_d$d.log 2>&1
done
