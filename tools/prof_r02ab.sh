export SHAPES="16,64,56,64,3,1;64,64,224,64,3,1;64,128,112,128,3,1;64,256,56,256,3,1;64,512,28,512,3,1;64,512,14,512,3,1;128,96,27,256,5,2;128,256,13,384,3,1;256,128,28,256,1,0,2"
for i in 1 2; do
timeout 600 python tools/shape_times.py > gpurun_out/r02ab_new$i.log 2>&1
FTC_LIB_PATH=build/variants/old.so timeout 600 python tools/shape_times.py > gpurun_out/r02ab_old$i.log 2>&1
done
FAULT_REPS=5 timeout 600 python tools/fault_one.py > gpurun_out/r02ab_fault.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ab_fault_launches.csv env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/r02ab_fault_ncu.log 2>&1
