for G in 1 2 3 4; do
  echo "G=$G  $(FTC_TC_DRAIN_CHUNKS=$G python tools/tc_time.py)"
  echo "      $(FTC_TC_DRAIN_CHUNKS=$G python tools/tc_acc.py)"
done
