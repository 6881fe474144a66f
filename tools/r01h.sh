python tools/glue_bench.py > gpurun_out/r01h_glue.log 2>&1
for v in "base:" "nofused:FTC_NO_FUSED=1"; do
  tag=${v%%:*}; e=${v#*:}
  env TAG=$tag $e python tools/layer_times.py >> gpurun_out/r01h_layers.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -k "glue or fused or net" > gpurun_out/r01h_pytest.log 2>&1; tail -3 gpurun_out/r01h_pytest.log
cat gpurun_out/r01h_glue.log gpurun_out/r01h_layers.log
