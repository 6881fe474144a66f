for G in 1 4 16 1000; do
  echo "G=$G full    $(FTC_TC_DRAIN_CHUNKS=$G python tools/tc_time.py)"
  echo "G=$G nothing $(FTC_TC_DEBUG=31 FTC_TC_DRAIN_CHUNKS=$G python tools/tc_time.py)"
  echo "G=$G mmaonly $(FTC_TC_DEBUG=23 FTC_TC_DRAIN_CHUNKS=$G python tools/tc_time.py)"
done
for G in 8 16 1000; do echo "G=$G acc $(FTC_TC_DRAIN_CHUNKS=$G python tools/tc_acc.py)"; done
