# r01f profiles (conv MMA order with B reuse): GPU tests, bench lines for every BASELINE
# config, the timed-region launch lists, ncu --set full of the 5 AlexNet convs
set -e
PFX=${PFX:-r01f}
python -m pytest tests -m gpu -q > gpurun_out/${PFX}_pytest.log 2>&1 || true
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${PFX}_smoke.log 2>&1
python bench.py > gpurun_out/${PFX}_alex.json 2> gpurun_out/${PFX}_alex.err
python bench.py --workload config1 --no-cpu-baseline > gpurun_out/${PFX}_c1.json 2> gpurun_out/${PFX}_c1.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${PFX}_ref.json 2> gpurun_out/${PFX}_ref.err
for w in vgg19 resnet18 yolov2; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${PFX}_$w.json 2> gpurun_out/${PFX}_$w.err
done
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${PFX}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${PFX}_ncu.log 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${PFX}_c1_launches.csv \
    python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${PFX}_ncu_c1.log 2>&1
python tools/alex_convs.py > gpurun_out/${PFX}_alexconvs.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 20 -c 5 -o gpurun_out/${PFX}_convs python tools/alex_convs.py > gpurun_out/${PFX}_ncu_convs.log 2>&1
tail -1 gpurun_out/${PFX}_pytest.log; cat gpurun_out/${PFX}_alex.json gpurun_out/${PFX}_c1.json gpurun_out/${PFX}_ref.json; tail -1 gpurun_out/${PFX}_smoke.log
