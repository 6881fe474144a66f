python tools/glue_bench.py > gpurun_out/r01g_glue.log 2>&1
for v in "base:" "nofused:FTC_NO_FUSED=1" "noatom:FTC_TC_DEBUG=4096" "noco5:FTC_TC_DEBUG=8192" "neither:FTC_TC_DEBUG=12288"; do
  tag=${v%%:*}; e=${v#*:}
  env TAG=$tag $e python tools/layer_times.py >> gpurun_out/r01g_layers.log 2>&1
done
cat gpurun_out/r01g_glue.log gpurun_out/r01g_layers.log
