for v in base cd32 cd8; do
  if [ $v = base ]; then L=""; else L="build/variants/$v.so"; fi
  FTC_LIB_PATH=$L ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r01aj_$v.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "$v: $(python tools/launches_table.py gpurun_out/r01aj_$v.csv 3 | grep cd1_parts)"
done
