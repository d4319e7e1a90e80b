# parity suite, quick benches cfg3/4/5, batch-tail sums
set -x
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
for CFG in ${CFGS:-3 4 5}; do
  env ${ENVS:-X=1} timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('cfg$CFG', round(d['value']/1e6,2), 'M nets/s', round(d['ms_per_step'],2), 'ms', {k:round(v,2) for k,v in d['roofline_step']['kernel_ms_per_step'].items()})"
  env ${ENVS:-X=1} DIAG_BATCHMAX=1 timeout 600 python tools/diag.py --config $CFG --reps 0 2>&1 | grep -E "sum of batch|max-latency"
done
