set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
for w in vgg19 resnet18 yolov2; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_$w.json 2> gpurun_out/r02a_bench_$w.err
done
