# Summaries under profiles/ from what tools/prof_r02_final2.sh left in gpurun_out/ (PFX=r02x):
# launch-list tables, ncu --set full tables, logs, bench lines and the conv traffic JSONs.
P=${PFX:?set PFX}
{
echo "# $P timed-step launch lists (ncu gpu__time_duration + DRAM bytes, --clock-control none, NVTX range timed_step, 2 steps)"
echo
echo "Command: \`ncu --nvtx --nvtx-include timed_step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --workload W --steps 2 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0\` (tools/prof_r02_final2.sh).  ncu serialises launches and flushes caches: per-launch times are cold-cache; the kernel SHARE of the step is what matches the bench."
for w in vgg19 config1 alexnet resnet18 yolov2; do echo; echo "## $w"; echo; python tools/launches_table.py gpurun_out/${P}_launches_$w.csv 2; done
echo; echo "## one faulted AlexNet-conv2 layer (tools/fault_one.py, FAULT_REPS=1: clean, CoC, RC, ClC calls)"; echo; python tools/launches_table.py gpurun_out/${P}_fault_launches.csv 1
} > profiles/${P}_bench_launches.md
{
echo "# $P ncu --set full: the tcgen05 convs of one protected step (VGG-19 b64, ResNet-18 b256, YOLOv2 b64), the HBM glue / staging / detect kernels (VGG-19) and the config-1 layer"
echo
echo "Captured with \`ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed_step/ -k regex:K\` on one bench step (tools/prof_r02_final2.sh), exported with \`ncu -i rep --page raw --csv\`; tables by tools/ncu_table.py.  L2 throughput % is against ncu's nominal LTS peak; the measured full-chip cap is about half of it (~6300 B/clk, B300_MICROARCH.md), so 43% here is ~85% of what the L2 delivers."
for k in vgg_convs resnet_convs yolo_convs vgg_glue config1; do echo; echo "## $k"; echo; python tools/ncu_table.py gpurun_out/${P}_${k}_raw.csv; done
} > profiles/${P}_ncu_full.md
cp gpurun_out/${P}_pytest.log profiles/${P}_pytest_gpu.log
cp gpurun_out/${P}_smoke.log profiles/${P}_smoke.log
cp gpurun_out/${P}_bench.json profiles/${P}_bench_vgg19.json
cp gpurun_out/${P}_ref.json profiles/${P}_bench_reference.json
cp gpurun_out/${P}_fault.log profiles/${P}_fault_times.log
for n in vgg19:vgg resnet18:resnet yolov2:yolo; do
  python tools/traffic_json.py ${n%%:*} gpurun_out/${P}_${n##*:}_convs_raw.csv profiles/${P}_ncu_full.md
done
