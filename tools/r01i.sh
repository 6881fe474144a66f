ncu --set full --clock-control none --import-source on -k regex:k_glue_tile -s 3 -c 1 -o gpurun_out/r01i_glue_pool1_v2ws python tools/glue_bench.py pool1 > gpurun_out/r01i_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_glue_tile -s 13 -c 1 -o gpurun_out/r01i_glue_pool1_v2 python tools/glue_bench.py pool1 > gpurun_out/r01i_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_act_pool_t -s 23 -c 1 -o gpurun_out/r01i_glue_pool1_legacy python tools/glue_bench.py pool1 > gpurun_out/r01i_ncu3.log 2>&1
tail -2 gpurun_out/r01i_ncu*.log
