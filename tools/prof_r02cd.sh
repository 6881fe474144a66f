set -x
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_conv_tc|k_co5|k_detect" --log-file gpurun_out/r02cd_diag.csv python tools/c4_diag2.py > gpurun_out/r02cd_diag.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/r02cd_bench.json 2> gpurun_out/r02cd_bench.err
echo done
