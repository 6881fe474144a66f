# restored-state check: GPU suite, short bench, and a shape sweep around the slow VGG layers
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02ca_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ca_pytest.log
SHAPES="64,128,112,128,3,1;32,128,112,128,3,1;64,128,56,128,3,1;64,128,112,256,3,1;64,64,112,128,3,1;64,256,112,128,3,1;64,64,224,64,3,1;64,64,224,128,3,1;64,256,56,256,3,1;64,128,56,256,3,1;256,128,28,128,3,1" timeout 600 python tools/shape_times.py > gpurun_out/r02ca_shapes.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/r02ca_bench.json 2> gpurun_out/r02ca_bench.err
echo done
