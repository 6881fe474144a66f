set -x
M="--metrics gpu__time_duration.sum --clock-control none --csv"
for dbg in 0 4096 8192 12288; do
FTC_TC_DEBUG=$dbg timeout 900 ncu $M -k regex:"k_conv_tc" --log-file gpurun_out/r02cc_dbg$dbg.csv python tools/c4_diag2.py > gpurun_out/r02cc_dbg$dbg.log 2>&1
done
echo done
