# batch-span vs slowest-net diagnostics (tracing) for the group path and the warp path
for CFG in ${CFGS:-3 5}; do for G in 1 0; do
  echo "=== cfg$CFG GAPLA_GROUP=$G"
  GAPLA_GROUP=$G DIAG_BATCHMAX=1 timeout 600 python tools/diag.py --config $CFG --reps 2 2>&1 | tail -16
done; done
