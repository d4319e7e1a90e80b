for CFG in ${CFGS:-3}; do for G in 1 0; do
  echo "=== cfg$CFG GAPLA_GROUP=$G"
  GAPLA_GROUP=$G DIAG_PERNET=1 timeout 600 python tools/diag.py --config $CFG --reps 0 2>&1 | tail -14
done; done
