S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $S --tool $tool --target-processes all --print-limit 20 python tools/sanitize.py > gpurun_out/r02ah_san_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/r02ah_san_$tool.log
done
