for G in 1 2 4; do echo "G=$G nhwc $(FTC_TC_DRAIN_CHUNKS=$G python tools/tc_time.py 2>&1)"; echo "G=$G nchw $(FTC_TC_NCHW=1 FTC_TC_DRAIN_CHUNKS=$G python tools/tc_time.py 2>&1)"; done
for G in 2 3; do echo "G=$G tests: $(FTC_TC_DRAIN_CHUNKS=$G timeout 300 python -m pytest tests/test_gpu_nets.py tests/test_golden.py -m gpu -q 2>&1 | grep -E 'passed|failed|AssertionError: \(' | head -5)"; done
