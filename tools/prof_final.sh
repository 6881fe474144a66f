set -e
python bench.py > gpurun_out/fin_alex.json 2> gpurun_out/fin_alex.err
python bench.py --workload config1 > gpurun_out/fin_c1.json 2> gpurun_out/fin_c1.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu.log 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/fin_c1_launches.csv \
    python bench.py --workload config1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_c1.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
cat gpurun_out/fin_alex.json gpurun_out/fin_c1.json gpurun_out/fin_ref.json; tail -2 gpurun_out/fin_smoke.log
