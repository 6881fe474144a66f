# A/B of a conv change: parity tests, tile trace, in-net kernel durations (ncu), short bench
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_determinism.py tests/test_gpu_nets.py -m gpu -q -x > gpurun_out/${PFX}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${PFX}_pytest.log
timeout 300 python tools/tc_trace3.py > gpurun_out/${PFX}_trace_c3.log 2>&1
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_conv_tc|k_co5|k_detect" --log-file gpurun_out/${PFX}_diag.csv python tools/c4_diag2.py > gpurun_out/${PFX}_diag.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_bench.json 2> gpurun_out/${PFX}_bench.err
echo done
