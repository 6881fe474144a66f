timeout 300 python tools/seq_time.py > gpurun_out/r02ae_base.log 2>&1
for v in seq_16_8 seq_16_16 seq_8_16 old; do FTC_LIB_PATH=build/variants/$v.so timeout 300 python tools/seq_time.py > gpurun_out/r02ae_$v.log 2>&1; done
