set -x
for d in 16 17 24 28 29 30 31 13 14; do
FTC_TC_DEBUG=$d timeout 600 python tools/layer_times.py > gpurun_out/r02o_d$d.log 2>&1
done
