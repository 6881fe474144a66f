set -x
timeout 900 python -m pytest tests/test_gpu_nets.py tests/test_abi_symbols.py -m gpu -q -x > gpurun_out/${PFX}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${PFX}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 2 > gpurun_out/${PFX}_bench.json 2> gpurun_out/${PFX}_bench.err
FTC_NO_ELIDE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_bench_noelide.json 2> gpurun_out/${PFX}_bench_noelide.err
echo done
