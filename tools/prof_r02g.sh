FTC_NO_PDL=1 python tools/determinism.py > gpurun_out/r02g_det_nopdl.log 2>&1
python tools/determinism.py > gpurun_out/r02g_det.log 2>&1
FTC_NO_PDL=1 FTC_LIB_PATH=build/variants/commit1.so python tools/determinism.py > gpurun_out/r02g_det_commit1_nopdl.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --campaign-runs 0 --no-cpu-baseline > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
FTC_LIB_PATH=build/variants/commit1.so timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --campaign-runs 0 --no-cpu-baseline > gpurun_out/r02g_bench_commit1.json 2> gpurun_out/r02g_bench_commit1.err
