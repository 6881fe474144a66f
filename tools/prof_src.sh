# ncu source-level stall samples of one conv (SHAPES = one shape): where the epilogue's tile end waits
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -c 1 -o /tmp/convsrc python tools/shape_times.py > gpurun_out/${PFX}_ncu.log 2>&1
ncu -i /tmp/convsrc.ncu-rep --page source --csv > gpurun_out/${PFX}_source.csv 2>/dev/null
ncu -i /tmp/convsrc.ncu-rep --page details > gpurun_out/${PFX}_details.txt 2>/dev/null
echo done
