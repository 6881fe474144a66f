set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seq_sums567_staged -c 2 -o /tmp/seq env FAULT_REPS=1 python tools/fault_one.py > gpurun_out/r02cm_ncu.log 2>&1
ncu -i /tmp/seq.ncu-rep --page raw --csv > gpurun_out/r02cm_seq_raw.csv 2>/dev/null
ncu -i /tmp/seq.ncu-rep --page source --csv > gpurun_out/r02cm_seq_source.csv 2>/dev/null
ncu -i /tmp/seq.ncu-rep --page details > gpurun_out/r02cm_seq_details.txt 2>/dev/null
echo done
