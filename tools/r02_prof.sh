# ncu of a mid-run cfg5 k_assign launch + batch-tail diagnostics (sum of per-batch slowest-net latency)
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s ${SKIP:-40} -c 1 \
    -o gpurun_out/prof5 python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/ncu5.log 2>&1
tail -n 1 gpurun_out/ncu5.log
for CFG in ${CFGS:-3 4 5}; do
  echo "== cfg$CFG"; DIAG_BATCHMAX=1 timeout 600 python tools/diag.py --config $CFG --reps 0 2>&1 | grep -E "batches|max-latency"
done
DIAG_PERNET=1 timeout 600 python tools/diag.py --config 5 --reps 0 2>&1 | tail -11
