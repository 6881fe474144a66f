# r02 evidence: GPU suite, smoke, bench (VGG-19 headline + extras), reference arm, timed-step
# launch lists (VGG, config 1, AlexNet), ncu --set full of the convs of one step of every
# net and of the HBM glue / staging / detect kernels, the faulted-layer launch list.
PFX=${PFX:-r02}
set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${PFX}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${PFX}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${PFX}_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${PFX}_bench.json 2> gpurun_out/${PFX}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${PFX}_ref.json 2> gpurun_out/${PFX}_ref.err
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
B="--steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0"
for w in vgg19 config1 alexnet resnet18 yolov2; do
  timeout 900 ncu --nvtx --nvtx-include "timed_step/" $M --log-file gpurun_out/${PFX}_launches_$w.csv python bench.py --workload $w $B > gpurun_out/${PFX}_ncu_$w.log 2>&1
done
F="--set full --clock-control none --import-source on --nvtx --nvtx-include timed_step/"
timeout 1500 ncu $F -k regex:k_conv_tc -c 16 -o gpurun_out/${PFX}_vgg_convs python bench.py --workload vgg19 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_ncuf_vgg.log 2>&1
timeout 1500 ncu $F -k regex:k_conv_tc -c 20 -o gpurun_out/${PFX}_resnet_convs python bench.py --workload resnet18 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_ncuf_resnet.log 2>&1
timeout 1500 ncu $F -k regex:k_conv_tc -c 21 -o gpurun_out/${PFX}_yolo_convs python bench.py --workload yolov2 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_ncuf_yolo.log 2>&1
timeout 900 ncu $F -k regex:"k_act_pool|k_cd1|k_nhwc|k_detect|k_co5" -c 12 -o gpurun_out/${PFX}_vgg_glue python bench.py --workload vgg19 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_ncuf_glue.log 2>&1
timeout 900 ncu $F -c 3 -o gpurun_out/${PFX}_config1 python bench.py --workload config1 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_ncuf_c1.log 2>&1
FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/${PFX}_fault.log 2>&1
timeout 900 ncu $M --log-file gpurun_out/${PFX}_fault_launches.csv env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/${PFX}_fault_ncu.log 2>&1
echo done
