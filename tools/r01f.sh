python tools/glue_bench.py > gpurun_out/r01f_glue.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_glue_tile -s 3 -c 1 -o gpurun_out/r01f_glue_relu3 python tools/glue_bench.py relu3 > gpurun_out/r01f_ncu.log 2>&1
cat gpurun_out/r01f_glue.log
