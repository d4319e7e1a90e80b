# parity on the default build, then quick benches + per-size latency of alternate builds (GAPLA_SO)
set -x
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -5
for SO in ${SOS:-libgapla.so}; do
for CFG in ${CFGS:-3 5}; do
  GAPLA_SO=$SO timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline > gpurun_out/b_${SO}_$CFG.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b_${SO}_$CFG.json'));print('$SO cfg$CFG', round(d['value']/1e6,2), 'M nets/s', round(d['ms_per_step'],2), 'ms', d['roofline_step']['kernel_ms_per_step'])"
done
GAPLA_SO=$SO DIAG_PERNET=1 timeout 600 python tools/diag.py --config 3 --reps 0 2>&1 | tail -11
done
