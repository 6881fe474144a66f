for v in head g16 x8; do
  FTC_LIB_PATH=build/variants/$v.so TAG=$v python tools/layer_times.py >> gpurun_out/r01q_layers.log 2>&1
done
for v in head g16 x8; do
  FTC_LIB_PATH=build/variants/$v.so TAG=$v python tools/layer_times.py >> gpurun_out/r01q_layers.log 2>&1
done
cat gpurun_out/r01q_layers.log
