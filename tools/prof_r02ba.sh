# L2 strip test (is the long-K conv L2-bound?) and the CTA-pair B-multicast conv
set -x
S="64,256,56,256,3,1;64,512,28,512,3,1;64,128,112,128,3,1;64,64,224,64,3,1;64,512,14,512,3,1"
for d in 0 1 16 17 2 3 4 8 12 13 29 31; do
  echo "== FTC_TC_DEBUG=$d"; FTC_TC_DEBUG=$d SHAPES="$S" timeout 300 python tools/shape_times.py
done
echo "== CL2 check"
timeout 600 python tools/cl2_check.py && FTC_TC_CL=2 timeout 600 python tools/cl2_check.py
echo "== CL2 times"
FTC_TC_CL=2 SHAPES="$S" timeout 300 python tools/shape_times.py
SHAPES="$S" timeout 300 python tools/shape_times.py
echo "== bench vgg CL2"
FTC_TC_CL=2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --campaign-runs 0
echo "== traces"
TRACE_SHAPE="64,256,56,256,3,1" timeout 300 python tools/tc_trace2.py
TRACE_SHAPE="64,64,224,64,3,1" timeout 300 python tools/tc_trace2.py
TRACE_SHAPE="64,128,112,128,3,1" timeout 300 python tools/tc_trace2.py
echo "== split variants"
for v in split1 split2; do
  echo "-- $v"; FTC_LIB_PATH=build/variants/$v.so SHAPES="$S" timeout 300 python tools/shape_times.py
  FTC_LIB_PATH=build/variants/$v.so timeout 300 python tools/tc_check.py | tail -4
done
