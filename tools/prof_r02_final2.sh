# r02 evidence: GPU suite, smoke, bench (VGG-19 headline + extras), reference arm, timed-step
# launch lists (VGG, config 1, AlexNet), ncu --set full of the convs of one step of every
# net and of the HBM glue / staging / detect kernels, the faulted-layer launch list.
PFX=${PFX:-r02e}
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
# --set full reports are exported to CSV (raw page) and deleted: a GPU call brings back
# at most 64 MiB of gpurun_out/; the config-1 report (3 kernels) is kept whole
R=/tmp/ncurep; mkdir -p $R
full() {  # name, kernel regex, count, workload
  timeout 1500 ncu $F -f -k regex:"$2" -c $3 -o $R/$1 python bench.py --workload $4 --steps 1 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0 > gpurun_out/${PFX}_ncuf_$1.log 2>&1
  ncu -i $R/$1.ncu-rep --page raw --csv > gpurun_out/${PFX}_$1_raw.csv 2>/dev/null
}
full vgg_convs k_conv_tc 16 vgg19
full resnet_convs k_conv_tc 20 resnet18
full yolo_convs k_conv_tc 21 yolov2
full vgg_glue "k_act_|k_cd1|k_nhwc|k_detect|k_co5" 40 vgg19
full config1 "k_" 3 config1
cp $R/config1.ncu-rep gpurun_out/${PFX}_config1.ncu-rep
FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/${PFX}_fault.log 2>&1
timeout 900 ncu $M --log-file gpurun_out/${PFX}_fault_launches.csv env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/${PFX}_fault_ncu.log 2>&1
echo done
